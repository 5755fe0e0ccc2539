// probe.cu — C-ABI of the B200-native PROBE MoE hot path (see include/probe.h).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/probe.h"
#include "kernels.cuh"
#include "distill.cuh"
#include "sgemm_f32.cuh"

using namespace probe;

namespace {

// ----------------------------------------------------------------------------- errors
std::mutex g_err_mu;
std::string g_last_error;

probe_status fail(probe_ctx ctx, probe_status st, const char* fmt, ...);

// ----------------------------------------------------------------------------- TMA encode
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled g_encode = nullptr;

bool load_encode() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = reinterpret_cast<PFN_encodeTiled>(fn);
  return true;
}

// 2-D bf16 K-major operand map: dims {cols (K), rows}, box {64, box_rows}, SWIZZLE_128B, OOB → 0.
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  if (!load_encode()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor-map cache with STABLE addresses (fixed ring; a call uses <= 6 maps, so a
// returned pointer stays valid for the rest of that call and the next 250 encodes).
// fp32 output map for TMA tensor stores: box {32 cols (128 B), 32 rows}, SWIZZLE_128B.
bool make_map_f32_out(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  if (!load_encode()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp16 output map for TMA tensor stores: box {32 cols (64 B), 32 rows}, SWIZZLE_64B.
bool make_map_f16_out(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, bool wide = false) {
  if (!load_encode()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {wide ? 64u : 32u, 32};   // wide: 128-byte rows (epi_chunk64_f16, tma_out == 2)
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bf16 output map for TMA tensor stores (the SwiGLU / SiLU activations): box {32 cols (64 B),
// 32 rows}, SWIZZLE_64B — the same staging layout as the fp16 Y map.
bool make_map_bf16_out(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  if (!load_encode()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct MapCache {
  struct Ent {
    const void* p = nullptr;
    uint64_t rows = 0, cols = 0;
    uint32_t box = 0;
    CUtensorMap map;
  };
  static constexpr int kCap = 256;
  Ent ents[kCap];
  int next = 0;
  const CUtensorMap* get(const void* p, uint64_t rows, uint64_t cols, uint32_t box) {
    for (auto& e : ents)
      if (e.p == p && e.rows == rows && e.cols == cols && e.box == box) return &e.map;
    Ent& e = ents[next];
    next = (next + 1) % kCap;
    e.p = nullptr;
    if (!make_map(&e.map, p, rows, cols, box)) return nullptr;
    e.p = p; e.rows = rows; e.cols = cols; e.box = box;
    return &e.map;
  }
};

size_t al(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }
// bytes per element of activations / weights / Y: 2 (bf16 path; Y fp16, D2) or 4 (PROBE_FP32)
size_t esz(const probe_config& c) { return c.dtype == PROBE_FP32 ? 4 : 2; }

struct Scratch {
  size_t sym, logits, pprior, pres, pact, ids, gw, pos, hist, cbase, route, pred_local;
  size_t quota[2], reps[2], stats[2], pfctr[2], pids[2];
  size_t split_cum, slot_of, src_off, group_rows, reps_used;
  size_t s_g1, s_g2, s_gate, s_p1, s_p2, flags, win_t0, act, total;
  size_t gprior[2], gact[2], wcat, s_gp;   // fused gate + predictor stage 1 (by predicted-layer parity)
};

Scratch scratch_layout(const probe_config& c) {
  Scratch s{};
  const size_t G = c.ep_size, GL = c.local_ranks, E = c.num_experts, k = c.top_k, T = c.max_tokens;
  const size_t h = c.res_hidden > 0 ? c.res_hidden : 8, F = c.ffn, cap = c.recv_capacity;
  const size_t NC = (T + kChunk - 1) / kChunk, EL = E / G, S = EL + kMaxRb;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += al(bytes); return r; };
  s.sym = take(PROBE_NSYM * G * 8);
  s.logits = take(GL * T * E * 4);
  s.pprior = take(GL * T * E * 4);
  s.pres = take(GL * T * E * 4);
  s.pact = take(GL * T * h * esz(c));
  s.ids = take(GL * T * k * 4);
  s.gw = take(GL * T * k * 4);
  s.pos = take(GL * T * k * 4);
  s.hist = take(GL * NC * E * 4);
  s.cbase = take(GL * NC * E * 4);
  s.route = take(GL * T * k * 8);
  s.pred_local = take(GL * E * 4);
  for (int p = 0; p < 2; ++p) {
    s.quota[p] = take(G * E * G * 4);
    s.reps[p] = take(G * kMaxRb * 4);
    s.stats[p] = take(8 * 8);
    s.pfctr[p] = take(16);
    s.pids[p] = take(c.predispatch ? GL * T * k * 4 : 16);   // predicted top-k sets (NEXT-4)
  }
  s.split_cum = take(G * E * G * 4);
  s.slot_of = take(G * E * 4);
  s.src_off = take(G * S * G * 4);
  s.group_rows = take(G * S * 4);
  s.reps_used = take(G * kMaxRb * 4);
  s.s_g1 = take(sizeof(GemmSched));
  s.s_g2 = take(sizeof(GemmSched));
  s.s_gate = take(sizeof(GemmSched));
  s.s_p1 = take(sizeof(GemmSched));
  s.s_p2 = take(sizeof(GemmSched));
  s.flags = take(256);
  s.win_t0 = take(64);
  s.act = take(GL * cap * F * esz(c));
  // fused gate + predictor stage 1: prior logits and activation double-buffered by the parity of
  // the predicted layer (gate(L+1) on the main stream may run while predict(L+1) still reads them)
  const bool gp = c.fuse_gate_predictor != 0;
  for (int p = 0; p < 2; ++p) {
    s.gprior[p] = take(gp ? GL * T * E * 4 : 16);
    s.gact[p] = take(gp ? GL * T * h * 2 : 16);
  }
  s.wcat = take(gp ? (2 * E + h) * c.hidden * 2 : 16);
  s.s_gp = take(gp ? sizeof(GemmSched) : 16);
  s.total = al(o, 1024);
  return s;
}

void sym_sizes(const probe_config& c, uint64_t b[PROBE_NBUF]) {
  const uint64_t cap = c.recv_capacity, H = c.hidden, F = c.ffn, G = c.ep_size, E = c.num_experts;
  const uint64_t es = esz(c);
  b[PROBE_BUF_RECV] = al(cap * H * es, 1024);
  b[PROBE_BUF_Y] = al(cap * H * es, 1024);   // fp16 (D2) / fp32
  b[PROBE_BUF_REP_W13] = al(2 * kMaxRb * 2 * F * H * es, 1024);
  b[PROBE_BUF_REP_W2] = al(2 * kMaxRb * H * F * es, 1024);
  b[PROBE_BUF_BOARD] = al(4 * G * E * 4 + 1024, 1024);   // + int64 [G] measured windows (R26)
  b[PROBE_BUF_SIGNAL] = 4096;
  // dedup wire (§8(a) a6/a8): per-receive-row meta records and the source-side partial rows
  const uint64_t KQ = static_cast<uint64_t>(c.top_k < c.ep_size ? c.top_k : c.ep_size);
  b[PROBE_BUF_META] = c.dedup_wire ? al(cap * 16, 1024) : 1024;
  b[PROBE_BUF_COMB] = c.dedup_wire ? al(static_cast<uint64_t>(c.max_tokens) * KQ * H * es, 1024) : 1024;
  b[PROBE_BUF_PRE] = c.predispatch ? al(static_cast<uint64_t>(G) * c.max_tokens * H * es, 1024) : 1024;
  b[PROBE_BUF_SCRATCH] = scratch_layout(c).total;
}

}  // namespace

struct probe_ctx_s {
  probe_config cfg;
  Dims d;
  Scratch sl;
  uint8_t* scratch;
  std::vector<uint64_t> peer;   // host copy [NSYM][G]
  uint8_t* local_base[PROBE_NSYM];
  uint64_t sym_bytes[PROBE_NBUF];
  cudaStream_t aux = nullptr, pf = nullptr, pd = nullptr;   // pd: NEXT-4 pre-dispatch side stream
  cudaEvent_t ev_fwd_start = nullptr, ev_pd_done = nullptr;
  int pred_T[2] = {0, 0};
  cudaEvent_t ev_gate[2], ev_gemm[2], ev_comb[2], ev_pred[2], ev_plan[2], ev_slots[2], ev_disp[2];
  int aux_start = 0;     // PROBE_OPT_AUX_START: predictor(L+1) starts after gate(L) (0) or dispatch(L) (1)
  int l2hint = 0;        // PROBE_OPT_L2_HINTS: TMA L2 eviction hints of the expert GEMMs (LayoutIn::l2hint)
  bool pred_pair = true;  // PROBE_OPT_PRED_PAIR: the predictor's Ŵ1·x GEMM on CTA pairs
  int pred_maxreg = 0;   // PROBE_OPT_PRED_MAXREG: 192 ⇒ register-capped predictor GEMMs (a dispatch CTA fits beside)
  // CUDA-graph awareness: id of the stream capture each event was last recorded in (0 = eager)
  std::vector<std::pair<cudaEvent_t, unsigned long long>> ev_cap;
  int fwd_layer = -1000, pred_layer[2] = {-1000, -1000}, plan_layer[2] = {-1000, -1000},
      pf_layer[2] = {-1000, -1000};
  // fused gate + predictor stage 1: armed by probe_predict_prepare, done by the forward
  int gp_next = -1000;
  const void* gp_wn = nullptr;
  const void* gp_w1 = nullptr;
  struct GpDone { int layer = -1000; const void* x = nullptr; int T = 0; const void* wn = nullptr; const void* w1 = nullptr; };
  GpDone gp_done[2];
  int last_fwd_parity = 0;
  int last_T = 0;
  int num_sms = 148;
  int aux_sms = 74;   // grid cap for aux-stream (predictor) GEMMs: the main track keeps free SMs
  MapCache maps;
  CUtensorMap map_recv, map_act, map_rw13, map_rw2, map_y, map_act_out;
  std::string err;
  int64_t launches = 0;
  bool multi_process() const { return cfg.local_ranks != cfg.ep_size; }
  bool f32() const { return cfg.dtype == PROBE_FP32; }   // fp32 parity path (SIMT GEMMs)
  bool dbg_gemm2_repeat = false;   // PROBE_DEBUG_GEMM2_REPEAT=1 (analysis)
  int dbg_gap_us = 0;              // PROBE_DEBUG_GAP_US (analysis)
  bool unfused = false;   // PROBE_UNFUSED=1: logits written + separate top-k kernels (debug)
  bool ep_emulation = false;  // partition expert GEMMs by local rank (probe_set_option)
  bool fused_epi_topk = false;  // top-k in the GEMM epilogue instead of k_select (probe_set_option)
  bool pair_gemm = true;        // expert GEMMs on CTA pairs (cta_group::2); option turns it off
  bool y_wide = true;           // fp16 Y by 64-column TMA stores (PROBE_Y_WIDE=0 at init: 32-column, A/B)
  bool gemm2_512 = true;        // GEMM2 on 256×512 CTA-pair tiles (PROBE_G2_512=0 at init: 256×256, A/B)
  bool gemm1_512 = false;       // GEMM1 likewise (PROBE_G1_512=1 at init, A/B)
  bool g2_nb2 = true;           // GEMM2 256×512 with double-buffered wide stores (PROBE_G2_NB2=0 at init, A/B)
  // distillation workspace (NEXT-1), allocated on the first probe_distill_grad
  uint8_t* dbuf = nullptr;
  size_t dbytes = 0;
  // phase profiling: prof_max forwards × (PROBE_NPHASE + 1) timing events
  int prof_max = 0, prof_n = 0;
  std::vector<cudaEvent_t> prof_ev;
  cudaEvent_t pev(int ph) { return prof_ev[static_cast<size_t>(prof_n) * (PROBE_NPHASE + 1) + ph]; }
  bool profiling() const { return prof_n < prof_max; }
  template <class T>
  T* at(size_t off) const {
    return reinterpret_cast<T*>(scratch + off);
  }
};

namespace {

probe_status fail(probe_ctx ctx, probe_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_last_error = buf;
  if (ctx) ctx->err = buf;
  return st;
}

#define CK(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) return fail(ctx, PROBE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define CKL()                                                                                         \
  do {                                                                                                \
    ++ctx->launches;                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                              \
    if (e_ != cudaSuccess) return fail(ctx, PROBE_ECUDA, "launch @%d: %s", __LINE__, cudaGetErrorString(e_)); \
  } while (0)

// GEMM variants: (BN, STAGES, epilogue warps).  V_GATE: logits/predictor (N ≤ 256),
// V_SWIGLU: expert GEMM1 (bf16 act out), V_F32: expert GEMM2 (fp32 Y out, epilogue-heavy).
// GEMM variants: (BN, STAGES, epilogue warps).  V_128_6_4: router / predictor GEMMs (N ≤ 128),
// V_256_4_4: router GEMM for E > 128 (1-CTA), V_2CTA_256_6_4: the expert GEMMs on CTA pairs,
// V_256_4_4_EXP: the 1-CTA expert GEMMs for decode-sized groups, V_128_6_4_R192: register-capped
// predictor GEMMs (PROBE_OPT_PRED_MAXREG).  The numbering is the probe_bench_gemm `variant`
// argument; the other numbers were configurations measured slower in round 1 and removed.
enum GemmVariant { V_128_6_4 = 0, V_256_4_4 = 1, V_2CTA_256_6_4 = 6, V_256_4_4_EXP = 10, V_128_6_4_R192 = 11,
                   V_2CTA_128_8_4 = 12 /* CTA pair, 256×128 tiles, 8 stages: the predictor's N = E = 128 GEMM */,
                   V_2CTA_512_4_4 = 13 /* CTA pair, 256×512 tiles (one TMEM accumulator), 4 stages */,
                   V_2CTA_512_4_4_NB2 = 14 /* the same with double-buffered 64-column stores (≤ 384 groups) */ };

// Expert GEMMs leave registers for one 128-thread prefetch CTA per SM (a9 part 1 runs beside them):
// 256 × 224 + 128 × 48 = 62 K.  Splits that fill exactly 64 K (240 + 32, 232 + 48) did not
// co-reside (C2 part 1 stalled, 100 µs exposed wait), so 2 K registers stay free.
constexpr int kExpertMaxReg = 224;
static_assert(256 * kExpertMaxReg + 128 * kPrefetchPart1Reg <= 65536 - 2048, "part-1 prefetch CTA must fit");
// The 1-CTA expert GEMM (decode-sized groups, C2) keeps the lower cap 216: A/B at C2 on one
// box, 2 runs each: 216 → 1.53–1.54 M tok/s, part 1 pushes 95 of 119 MB, exposed wait 24 µs;
// 224 → 1.43 M tok/s, 71 MB, 110–118 µs.
#ifndef PROBE_EXP1_MAXREG
#define PROBE_EXP1_MAXREG 216
#endif
// ptxas at 216: the 1-CTA expert GEMM keeps a 48-byte stack (59 LDL/STL, C2 A/B above);
// at 255: 16 bytes.  Any override must still leave room for the part-1 prefetch CTA.
static_assert(256 * PROBE_EXP1_MAXREG + 128 * kPrefetchPart1Reg <= 65536 - 2048, "part-1 prefetch CTA must fit");

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel instance PER DEVICE (a
// process driving several devices must set it on each).
template <class K>
cudaError_t smem_attr_once(K kern, int bytes, uint64_t& done_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if ((done_mask >> (dev & 63)) & 1ull) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done_mask |= 1ull << (dev & 63);
  return e;
}

template <int BN, int ST, int EW, int NB = 1, int MAXR = 255>
cudaError_t launch_gemm_2cta(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1, const CUtensorMap& c,
                             const CUtensorMap& a2, GemmSched* s, int K, int K2, int grid, cudaStream_t st) {
  using L = Gemm2Smem<BN, ST, EW, NB>;
  static_assert(L::BYTES <= 232448, "shared memory budget");
  static uint64_t attr = 0;
  cudaError_t e = smem_attr_once(grouped_gemm_2cta_kernel<BN, ST, EW, MAXR, NB>, L::BYTES, attr);
  if (e != cudaSuccess) return e;
  grouped_gemm_2cta_kernel<BN, ST, EW, MAXR, NB><<<grid & ~1, 128 + 32 * EW, L::BYTES, st>>>(a, b0, b1, c, a2, s, K,
                                                                                             K2);
  return cudaGetLastError();
}

template <int BN, int ST, int EW, int NB = (EW == 8 ? 2 : 1), int MAXR = 255>
cudaError_t launch_gemm_t(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1, const CUtensorMap& c,
                          const CUtensorMap& a2, GemmSched* s, int K, int K2, int grid, cudaStream_t st) {
  using L = GemmSmem<BN, ST, EW, NB>;
  static_assert(L::BYTES <= 232448, "shared memory budget");
  static uint64_t attr = 0;
  cudaError_t e = smem_attr_once(grouped_gemm_kernel<BN, ST, EW, NB, MAXR>, L::BYTES, attr);
  if (e != cudaSuccess) return e;
  grouped_gemm_kernel<BN, ST, EW, NB, MAXR><<<grid, 128 + 32 * EW, L::BYTES, st>>>(a, b0, b1, c, a2, s, K, K2);
  return cudaGetLastError();
}

cudaError_t launch_gemm_v(int v, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                          const CUtensorMap& c, GemmSched* s, int K, int grid, cudaStream_t st,
                          const CUtensorMap* a2 = nullptr, int K2 = 0) {
  const CUtensorMap& A2 = a2 ? *a2 : a;
  switch (v) {
    case V_128_6_4: return launch_gemm_t<128, 6, 4>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_256_4_4: return launch_gemm_t<256, 4, 4>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_2CTA_256_6_4: return launch_gemm_2cta<256, 6, 4, 1, kExpertMaxReg>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_2CTA_512_4_4: return launch_gemm_2cta<512, 4, 4, 1, kExpertMaxReg>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_2CTA_512_4_4_NB2: return launch_gemm_2cta<512, 4, 4, 2, kExpertMaxReg>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_256_4_4_EXP: return launch_gemm_t<256, 4, 4, 1, PROBE_EXP1_MAXREG>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_128_6_4_R192: return launch_gemm_t<128, 6, 4, 1, 192>(a, b0, b1, c, A2, s, K, K2, grid, st);
    case V_2CTA_128_8_4: return launch_gemm_2cta<128, 8, 4, 1, kExpertMaxReg>(a, b0, b1, c, A2, s, K, K2, grid, st);
  }
  return cudaErrorInvalidValue;
}
int variant_bn(int v) {
  return (v == V_128_6_4 || v == V_128_6_4_R192 || v == V_2CTA_128_8_4)
             ? 128
             : ((v == V_2CTA_512_4_4 || v == V_2CTA_512_4_4_NB2) ? 512 : 256);
}
int variant_tm(int v) {
  return (v == V_2CTA_256_6_4 || v == V_2CTA_128_8_4 || v == V_2CTA_512_4_4 || v == V_2CTA_512_4_4_NB2) ? 256 : 128;
}
bool variant_ok(int v) {
  return v == V_128_6_4 || v == V_256_4_4 || v == V_2CTA_256_6_4 || v == V_256_4_4_EXP || v == V_128_6_4_R192 ||
         v == V_2CTA_128_8_4 || v == V_2CTA_512_4_4 || v == V_2CTA_512_4_4_NB2;
}

template <int BN>
cudaError_t launch_gemm(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1, GemmSched* s, int K,
                        int grid, cudaStream_t st) {
  return launch_gemm_v(BN == 256 ? V_256_4_4 : V_128_6_4, a, b0, b1, a, s, K, grid, st);
}

template <bool PRED>
cudaError_t launch_select(const Dims& d, int T, int nchunks, cudaStream_t st, const float* lg, const float* b,
                          int32_t* ids, float* gw, int32_t* pos, int32_t* hist, int32_t* cnt,
                          float* lo = nullptr, int32_t* pids = nullptr, const float* lg2 = nullptr) {
  const size_t smem = 0;
  dim3 grid(nchunks, d.GL);
#define SEL(KK)                                                                                         \
  case KK: {                                                                                            \
    k_select<KK, PRED><<<grid, 128, smem, st>>>(d, T, lg, b, ids, gw, pos, hist, cnt, lo, pids, lg2);  \
    break;                                                                                              \
  }
  switch (d.k) {
    SEL(1) SEL(2) SEL(3) SEL(4) SEL(5) SEL(6) SEL(7) SEL(8)
    default: return cudaErrorInvalidValue;
  }
#undef SEL
  return cudaGetLastError();
}

template <bool PRED>
void launch_topk(const Dims& d, int T, int nchunks, cudaStream_t st, const float* lg, const float* lg2, const float* b,
                 int32_t* ids, float* gw, int32_t* pos, int32_t* hist, int32_t* pc, float* lo) {
  dim3 grid(nchunks, d.GL);
  if (d.E <= 32) k_topk<1, PRED><<<grid, 128, 0, st>>>(d, T, lg, lg2, b, ids, gw, pos, hist, pc, lo);
  else if (d.E <= 64) k_topk<2, PRED><<<grid, 128, 0, st>>>(d, T, lg, lg2, b, ids, gw, pos, hist, pc, lo);
  else if (d.E <= 128) k_topk<4, PRED><<<grid, 128, 0, st>>>(d, T, lg, lg2, b, ids, gw, pos, hist, pc, lo);
  else k_topk<8, PRED><<<grid, 128, 0, st>>>(d, T, lg, lg2, b, ids, gw, pos, hist, pc, lo);
}

GemmGroup mk_group(int a_row, int m, int b_row, int b_sel, int mode, int n, int ldc, void* out) {
  GemmGroup g;
  g.a_row = a_row; g.m = m; g.b_row = b_row; g.b_sel = b_sel; g.mode = mode; g.n = n; g.ldc = ldc;
  g.tile_start = 0; g.out_row = 0; g.tma_out = 0; g.topk = 0; g.rows_per_rank = 1; g.k_off = 0; g.n_split = 0; g.out = out;
  g.aux = nullptr; g.bias = nullptr;
  return g;
}

Sym sym_of(probe_ctx ctx) { return Sym{ctx->at<const uint64_t>(ctx->sl.sym)}; }

unsigned long long capture_id(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(st, &cs, &id) != cudaSuccess) return 0;
  return cs == cudaStreamCaptureStatusActive ? id : 0;
}

cudaError_t ev_record(probe_ctx ctx, cudaEvent_t ev, cudaStream_t st) {
  cudaError_t e = cudaEventRecord(ev, st);
  const unsigned long long id = capture_id(st);
  for (auto& pr : ctx->ev_cap)
    if (pr.first == ev) { pr.second = id; return e; }
  ctx->ev_cap.emplace_back(ev, id);
  return e;
}

// A capturing stream never waits on an event recorded outside its own capture (illegal in
// a graph; the contract is that eager work is complete before capture begins).  A
// non-capturing stream waiting on a captured event is how the aux / prefetch streams fork
// into the graph.
cudaError_t ev_wait(probe_ctx ctx, cudaStream_t st, cudaEvent_t ev) {
  const unsigned long long cur = capture_id(st);
  if (cur != 0) {
    unsigned long long evid = 0;
    for (auto& pr : ctx->ev_cap)
      if (pr.first == ev) evid = pr.second;
    if (evid != cur) return cudaSuccess;
  }
  return cudaStreamWaitEvent(st, ev, 0);
}

enum { BAR_COUNTS = 0, BAR_DISPATCH = 1, BAR_Y = 2, BAR_PRED = 3, BAR_PREFETCH = 4 };
// scratch flags (int32 words): 0 device error word, 1 prefetch suspend flag, 2/3 prefetch
// part-1/part-2 KiB pushed, 4 static-EP fallbacks, kEpochSlot.. cross-process barrier epochs (one per kind)
constexpr int kEpochSlot = 16;
constexpr int kFallbackSlot = 4;   // layers whose plan would have overflowed → ran static EP
constexpr int kHitSlot = 5;        // NEXT-4: (token, dest) pairs pre-dispatched (hit) / shipped after the gate (miss)
static_assert(kEpochSlot + kSigKinds <= 64, "flags area is 256 bytes");

// fp32 parity path: grouped SIMT GEMM over a device-resident schedule (sgemm_f32.cuh)
cudaError_t launch_sgemm(probe_ctx ctx, const GemmSched* sc, const void* A, const void* B0, const void* B1, int K,
                         cudaStream_t st) {
  k_sgemm_grouped<<<ctx->num_sms * 4, 256, 0, st>>>(sc, static_cast<const float*>(A), static_cast<const float*>(B0),
                                                    static_cast<const float*>(B1), K);
  return cudaGetLastError();
}

// Cross-process barrier (no-op when this process hosts every rank: stream order suffices).
cudaError_t xbarrier(probe_ctx ctx, int kind, cudaStream_t st) {
  if (!ctx->multi_process()) return cudaSuccess;
  const Dims& d = ctx->d;
  // epochs live in device memory (flags[kEpochSlot + kind]) so graph replays advance them
  k_xbarrier<<<1, ((d.GL * d.G + 31) / 32) * 32, 0, st>>>(d, sym_of(ctx), PROBE_BUF_SIGNAL, kind,
                                                          reinterpret_cast<uint32_t*>(ctx->at<int32_t>(ctx->sl.flags) + kEpochSlot));
  ++ctx->launches;
  return cudaGetLastError();
}

}  // namespace

extern "C" {

probe_status probe_workspace(const probe_config* cfg, uint64_t bytes[PROBE_NBUF]) {
  if (!cfg || !bytes) return fail(nullptr, PROBE_EINVAL, "probe_workspace: null argument");
  sym_sizes(*cfg, bytes);
  return PROBE_OK;
}

static probe_status validate(const probe_config& c) {
  if (c.ep_size < 1 || c.ep_size > kMaxG) return fail(nullptr, PROBE_EINVAL, "ep_size %d out of [1,%d]", c.ep_size, kMaxG);
  if (c.local_ranks < 1 || c.rank_begin < 0 || c.rank_begin + c.local_ranks > c.ep_size)
    return fail(nullptr, PROBE_EINVAL, "local rank range [%d,%d) outside [0,%d)", c.rank_begin,
                c.rank_begin + c.local_ranks, c.ep_size);
  if (c.num_experts < 1 || c.num_experts > kMaxE || c.num_experts % c.ep_size)
    return fail(nullptr, PROBE_ESHAPE, "num_experts %d must be in [1,%d] and divisible by ep_size %d", c.num_experts,
                kMaxE, c.ep_size);
  if (c.top_k < 1 || c.top_k > c.num_experts || c.top_k > kMaxK)
    return fail(nullptr, PROBE_ESHAPE, "top_k %d out of range", c.top_k);
  if (c.hidden < 64 || c.hidden % 64 || c.ffn < 64 || c.ffn % 64)
    return fail(nullptr, PROBE_ESHAPE, "hidden %d and ffn %d must be positive multiples of 64", c.hidden, c.ffn);
  if (c.res_hidden < 0 || c.res_hidden % 8) return fail(nullptr, PROBE_ESHAPE, "res_hidden %d must be a multiple of 8", c.res_hidden);
  if (c.num_experts % 8) return fail(nullptr, PROBE_ESHAPE, "num_experts %d must be a multiple of 8", c.num_experts);
  if (c.max_tokens < 1 || c.recv_capacity < 1) return fail(nullptr, PROBE_EINVAL, "max_tokens/recv_capacity must be >= 1");
  // the local ranks' RECV / Y copies are one contiguous [local_ranks·cap, H] tensor for the GEMMs'
  // TMA maps: cap·H·sizeof(act) must be a multiple of the 1024-byte buffer stride (H % 64 == 0)
  if (c.recv_capacity % 8) return fail(nullptr, PROBE_EINVAL, "recv_capacity %d must be a multiple of 8", c.recv_capacity);
  if (c.dedup_wire != 0 && c.dedup_wire != 1) return fail(nullptr, PROBE_EINVAL, "dedup_wire %d not in {0, 1}", c.dedup_wire);
  if (c.predispatch != 0 && c.predispatch != 1) return fail(nullptr, PROBE_EINVAL, "predispatch %d not in {0, 1}", c.predispatch);
  if (c.predispatch && !c.dedup_wire) return fail(nullptr, PROBE_EINVAL, "predispatch requires dedup_wire = 1");
  if (c.fuse_gate_predictor != 0 && c.fuse_gate_predictor != 1)
    return fail(nullptr, PROBE_EINVAL, "fuse_gate_predictor %d not in {0, 1}", c.fuse_gate_predictor);
  if (c.fuse_gate_predictor && (c.dtype != PROBE_BF16 || c.num_experts % 32 || c.top_k > kTopkMax))
    return fail(nullptr, PROBE_ESHAPE, "fuse_gate_predictor needs bf16, E %% 32 == 0 and top_k <= %d", kTopkMax);
  if (static_cast<int64_t>(c.local_ranks) * c.recv_capacity > (1ll << 30) ||
      static_cast<int64_t>(c.local_ranks) * c.max_tokens > (1ll << 28))
    return fail(nullptr, PROBE_ECAPACITY, "capacity too large");
  if (c.replica_budget < 0 || c.replica_budget > kMaxRb)
    return fail(nullptr, PROBE_EBUDGET, "replica_budget %d out of [0,3] (P:476)", c.replica_budget);
  if (c.kmax < 0) return fail(nullptr, PROBE_EINVAL, "kmax < 0");
  if (c.n_sat < 0 || c.alpha_ps < 0 || c.beta_ps < 0 || c.bw_bytes_per_us < 0)
    return fail(nullptr, PROBE_EINVAL, "negative cost constant");
  if (c.dtype != PROBE_BF16 && c.dtype != PROBE_FP32) return fail(nullptr, PROBE_EINVAL, "dtype %d not in {0, 1}", c.dtype);
  if (c.expert_bytes != 3ll * c.hidden * c.ffn * static_cast<int64_t>(esz(c)))
    return fail(nullptr, PROBE_EINVAL, "expert_bytes %lld != 3*H*F*sizeof(dtype) = %lld", (long long)c.expert_bytes,
                3ll * c.hidden * c.ffn * static_cast<int64_t>(esz(c)));
  return PROBE_OK;
}

probe_status probe_init(const probe_config* cfg, const uint64_t* peer_ptrs, void* scratch, probe_ctx* out) {
  probe_ctx ctx = nullptr;
  if (!cfg || !peer_ptrs || !scratch || !out) return fail(nullptr, PROBE_EINVAL, "probe_init: null argument");
  probe_status st = validate(*cfg);
  if (st != PROBE_OK) return st;
  ctx = new probe_ctx_s();
  ctx->cfg = *cfg;
  const probe_config& c = *cfg;
  ctx->d = Dims{c.ep_size, c.rank_begin, c.local_ranks, c.num_experts, c.num_experts / c.ep_size, c.top_k,
                c.hidden, c.ffn, c.res_hidden, c.max_tokens, c.recv_capacity, c.replica_budget};
  ctx->sl = scratch_layout(c);
  {
    const char* u = getenv("PROBE_UNFUSED");
    ctx->unfused = u && u[0] == '1';
    // analysis only (GEMM2's in-layer rate): repeat GEMM2 inside its phase / idle gap before it
    const char* r2 = getenv("PROBE_DEBUG_GEMM2_REPEAT");
    ctx->dbg_gemm2_repeat = r2 && r2[0] == '1';
    const char* gap = getenv("PROBE_DEBUG_GAP_US");
    ctx->dbg_gap_us = gap ? atoi(gap) : 0;
  }
  ctx->scratch = static_cast<uint8_t*>(scratch);
  sym_sizes(c, ctx->sym_bytes);
  const int G = c.ep_size;
  ctx->peer.assign(peer_ptrs, peer_ptrs + PROBE_NSYM * G);
  for (int b = 0; b < PROBE_NSYM; ++b) {
    ctx->local_base[b] = reinterpret_cast<uint8_t*>(ctx->peer[b * G + c.rank_begin]);
    for (int l = 0; l < c.local_ranks; ++l) {
      const uint64_t want = ctx->peer[b * G + c.rank_begin] + static_cast<uint64_t>(l) * ctx->sym_bytes[b];
      if (ctx->peer[b * G + c.rank_begin + l] != want) {
        delete ctx;
        return fail(nullptr, PROBE_ECOMM, "buffer %d: local ranks must be contiguous with stride %llu", b,
                    (unsigned long long)ctx->sym_bytes[b]);
      }
    }
    for (int r = 0; r < G; ++r)
      if (ctx->peer[b * G + r] == 0 || ctx->peer[b * G + r] % 1024) {
        delete ctx;
        return fail(nullptr, PROBE_ECOMM, "buffer %d of rank %d null or not 1024-aligned", b, r);
      }
  }
  if (reinterpret_cast<uintptr_t>(scratch) % 1024) {
    delete ctx;
    return fail(nullptr, PROBE_EINVAL, "scratch must be 1024-byte aligned");
  }
  cudaError_t e = cudaMemcpy(ctx->scratch + ctx->sl.sym, ctx->peer.data(), PROBE_NSYM * G * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(ctx->scratch + ctx->sl.flags, 0, 256);
  if (e == cudaSuccess) e = cudaMemset(ctx->scratch + ctx->sl.s_g1, 0, sizeof(GemmSched));
  if (e == cudaSuccess) e = cudaMemset(ctx->scratch + ctx->sl.s_g2, 0, sizeof(GemmSched));
  // The aux track (predictor, planner) and the prefetch run on the highest-priority streams:
  // the block scheduler then hands them SMs as soon as main-track CTAs retire, so the plan
  // for L+1 is ready during dispatch(L) and prefetch part 1 can run beside the expert GEMMs
  // (with default priority the 8192 dispatch CTAs and then the persistent GEMM CTAs went
  // first, the planner — 32 KB of shared memory, no room beside a GEMM CTA — ran after
  // GEMM2, and part 1 found the combine's suspend flag already raised).
  int prio_lo = 0, prio_hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->pf, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->pd, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fwd_start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_pd_done, cudaEventDisableTiming);
  for (int p = 0; p < 2 && e == cudaSuccess; ++p) {
    cudaEvent_t* evs[7] = {&ctx->ev_gate[p], &ctx->ev_gemm[p], &ctx->ev_comb[p], &ctx->ev_pred[p], &ctx->ev_plan[p],
                           &ctx->ev_slots[p], &ctx->ev_disp[p]};
    for (auto* ev : evs)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  }
  int dev = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
  ctx->aux_sms = ctx->num_sms / 2;
  if (e == cudaSuccess) {
    const size_t split_smem = static_cast<size_t>(G) * c.num_experts * G * 4;   // k_layout's split [G][E][G]
    e = cudaFuncSetAttribute(k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(split_smem));
  }
  if (e != cudaSuccess) {
    delete ctx;
    return fail(nullptr, PROBE_ECUDA, "probe_init: %s", cudaGetErrorString(e));
  }
  const uint64_t GL = c.local_ranks, cap = c.recv_capacity, H = c.hidden, F = c.ffn;
  if (const char* yw = getenv("PROBE_Y_WIDE")) ctx->y_wide = yw[0] != '0';   // analysis A/B only
  if (const char* g5 = getenv("PROBE_G2_512")) ctx->gemm2_512 = g5[0] != '0';
  if (const char* g5 = getenv("PROBE_G1_512")) ctx->gemm1_512 = g5[0] != '0';
  if (const char* g5 = getenv("PROBE_G2_NB2")) ctx->g2_nb2 = g5[0] != '0';
  bool ok = make_map(&ctx->map_recv, ctx->local_base[PROBE_BUF_RECV], GL * cap, H, 128) &&
            make_map(&ctx->map_act, ctx->scratch + ctx->sl.act, GL * cap, F, 128) &&
            make_map(&ctx->map_rw13, ctx->local_base[PROBE_BUF_REP_W13], GL * 2 * kMaxRb * 2 * F, H, 128) &&
            make_map(&ctx->map_rw2, ctx->local_base[PROBE_BUF_REP_W2], GL * 2 * kMaxRb * H, F, 128) &&
            make_map_f16_out(&ctx->map_y, ctx->local_base[PROBE_BUF_Y], GL * cap, H, ctx->y_wide) &&
            (c.dtype == PROBE_FP32 || make_map_bf16_out(&ctx->map_act_out, ctx->scratch + ctx->sl.act, GL * cap, F));
  if (!ok) {
    delete ctx;
    return fail(nullptr, PROBE_ECUDA, "probe_init: cuTensorMapEncodeTiled failed");
  }
  *out = ctx;
  return PROBE_OK;
}

probe_status probe_moe_forward(probe_ctx ctx, int32_t layer, const void* x, int32_t T, const void* w_router,
                               const float* b_router, const void* w13, const void* w2, int32_t use_plan, void* out,
                               int32_t out_fp32, int32_t* topk_ids, float* topk_w, void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  if (!x || !w_router || !w13 || !w2 || !out) return fail(ctx, PROBE_EINVAL, "probe_moe_forward: null pointer");
  if (layer < 0) return fail(ctx, PROBE_EINVAL, "layer %d < 0", layer);
  if (T < 1 || T > ctx->cfg.max_tokens) return fail(ctx, PROBE_ECAPACITY, "T=%d outside [1, max_tokens=%d]", T, ctx->cfg.max_tokens);
  const int p = layer & 1;
  if (use_plan) {
    if (ctx->plan_layer[p] != layer) return fail(ctx, PROBE_ESTATE, "layer %d: use_plan without probe_plan(%d)", layer, layer);
    if (ctx->pf_layer[p] != layer)
      return fail(ctx, PROBE_ESTATE, "layer %d: use_plan without probe_prefetch(%d, START)", layer, layer);
  }
  const Dims& d0 = ctx->d;
  Dims d = d0;
  d.T = T;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t GL = d.GL, H = d.H, F = d.F, E = d.E;
  const int nchunks = (T + kChunk - 1) / kChunk;
  const bool f32 = ctx->f32();
  const CUtensorMap* mx = f32 ? nullptr : ctx->maps.get(x, GL * T, H, 128);
  const CUtensorMap* m13 = f32 ? nullptr : ctx->maps.get(w13, GL * d.EL * 2 * F, H, 128);
  const CUtensorMap* m2 = f32 ? nullptr : ctx->maps.get(w2, GL * d.EL * H, F, 128);
  if (!f32 && (!mx || !m13 || !m2)) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
  const Scratch& s = ctx->sl;
  int32_t* err = ctx->at<int32_t>(s.flags);
  int32_t* suspend = err + 1;
  const bool prof = ctx->profiling();
#define MARK(ph) \
  if (prof) CK(cudaEventRecord(ctx->pev(ph), st))
  MARK(0);
  // NEXT-4 pre-dispatch: this layer was predicted, so push every token's x row to the home
  // ranks of its predicted experts on a side stream while the gate below computes the routing
  const int row_bytes = static_cast<int>(H * esz(ctx->cfg));
  const bool predisp = ctx->cfg.predispatch && use_plan && ctx->pred_layer[p] == layer && ctx->pred_T[p] == T &&
                       !f32;
  if (predisp) {
    CK(ev_record(ctx, ctx->ev_fwd_start, st));
    CK(ev_wait(ctx, ctx->pd, ctx->ev_fwd_start));
    CK(ev_wait(ctx, ctx->pd, ctx->ev_plan[p]));     // predicted sets of this layer (predict → plan, aux)
    k_predispatch<<<(static_cast<int>(GL) * T + 7) / 8, 256, 0, ctx->pd>>>(
        d, T, ctx->cfg.max_tokens, static_cast<const uint8_t*>(x), row_bytes, ctx->at<int32_t>(s.pids[p]),
        sym_of(ctx), PROBE_BUF_PRE);
    CKL();
    if (prof) CK(cudaEventRecord(ctx->pev(PROBE_NPHASE - 1), ctx->pd));
    CK(ev_record(ctx, ctx->ev_pd_done, ctx->pd));
  } else if (prof) {
    CK(cudaEventRecord(ctx->pev(PROBE_NPHASE - 1), st));
  }
  // a1 gate: logits = x W_rᵀ on tcgen05 (fp32 logits by TMA stores, HBM-bound) → thread-per-token
  // select (top-k by sorting networks + softmax + dispatch ranks).  The GEMM-epilogue top-k
  // (EPI_TOPK, PROBE_OPT_FUSED_EPILOGUE_TOPK) saves the 2×33 MB logits round trip but measured
  // 20 µs slower at C1.
  const bool sel = d.k <= kTopkMax && d.E <= kMaxE && !ctx->unfused;
  const bool fused_gate = sel && ctx->fused_epi_topk && !f32;
  // fused gate + predictor stage 1 (probe_predict_prepare(layer+1) armed it): one GEMM over x for
  // [W_L ; W_{L+1} ; Ŵ1] → gate logits, prior logits of L+1, a = bf16(SiLU(Ŵ1 x)) (Eq. (P), R8)
  const bool gp = ctx->cfg.fuse_gate_predictor && ctx->gp_next == layer + 1 && sel && !fused_gate && !f32;
  const int gpp = (layer + 1) & 1;
  if (gp) {
    const uint64_t M = GL * T, h = d.h;
    const bool res = ctx->gp_w1 != nullptr;
    const uint64_t wrows = 2 * E + (res ? h : 0);
    const int64_t blk = static_cast<int64_t>(E * H * 2 / 16);
    const bool pairg = M >= 256;
    const CUtensorMap* mw = ctx->maps.get(ctx->scratch + s.wcat, wrows, H, 128);
    if (!mw) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
    CUtensorMap mact;
    const bool tma_act = res && h % 32 == 0 && make_map_bf16_out(&mact, ctx->scratch + s.gact[gpp], M, h);
    SmallGroups sg{};
    sg.BN = 256;
    sg.TM = pairg ? 256 : 128;
    sg.n = res ? 2 : 1;
    sg.g[0] = mk_group(0, static_cast<int>(M), 0, 0, EPI_F32, 2 * d.E, d.E, ctx->at<float>(s.logits));
    sg.g[0].n_split = d.E;
    sg.g[0].aux = ctx->at<float>(s.gprior[gpp]);
    if (res) {
      sg.g[1] = mk_group(0, static_cast<int>(M), 2 * d.E, 0, EPI_SILU_BF16, d.h, d.h, ctx->scratch + s.gact[gpp]);
      sg.g[1].tma_out = tma_act ? 1 : 0;
    }
    // ≤ 256 row chunks (≤ 512 groups), each a whole number of tiles
    const int TM = sg.TM;
    const int CM = static_cast<int>(((M + 255) / 256 + TM - 1) / TM * TM);
    k_gate_pred_prep<<<ctx->num_sms, 256, 0, st>>>(ctx->at<GemmSched>(s.s_gp), sg, static_cast<int>(M), CM,
                                                   ctx->at<uint4>(s.wcat), static_cast<const uint4*>(w_router), blk,
                                                   static_cast<const uint4*>(ctx->gp_wn), blk,
                                                   static_cast<const uint4*>(ctx->gp_w1),
                                                   res ? static_cast<int64_t>(h * H * 2 / 16) : 0);
    CKL();
    CK(launch_gemm_v(pairg ? V_2CTA_256_6_4 : V_256_4_4, *mx, *mw, *mw, tma_act ? mact : *mx,
                     ctx->at<GemmSched>(s.s_gp), d.H, ctx->num_sms, st));
    ctx->gp_done[gpp].layer = layer + 1;
    ctx->gp_done[gpp].x = x;
    ctx->gp_done[gpp].T = T;
    ctx->gp_done[gpp].wn = ctx->gp_wn;
    ctx->gp_done[gpp].w1 = ctx->gp_w1;
    ctx->gp_next = -1000;
  }
  SmallGroups sg{};
  sg.n = 1;
  sg.BN = d.E <= 128 ? 128 : 256;
  if (gp) {
    // logits already written by the fused GEMM above
  } else if (fused_gate) {
    sg.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_TOPK, d.E, d.E, ctx->at<int32_t>(s.ids));
    sg.g[0].topk = d.k;
    sg.g[0].aux = ctx->at<float>(s.gw);
    sg.g[0].bias = b_router;
  } else {
    sg.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.logits));
  }
  // fp32 logits by TMA tensor stores (full 32-row slabs; measured 60 vs 80 µs at C1 shapes)
  CUtensorMap mlog_f32;
  const bool gate_tma = !gp && !fused_gate && !f32 && d.E % 32 == 0 &&
                        make_map_f32_out(&mlog_f32, ctx->at<float>(s.logits), GL * T, E);
  if (gate_tma) sg.g[0].tma_out = 1;
  if (!gp) {
    k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_gate), sg);
    CKL();
  }
  if (gp) {
  } else if (f32) {
    CK(launch_sgemm(ctx, ctx->at<GemmSched>(s.s_gate), x, w_router, w_router, d.H, st));
  } else {
    const CUtensorMap* mr = ctx->maps.get(w_router, E, H, sg.BN / 2);
    if (!mr) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
    CUtensorMap mlog = *mx;
    CK(launch_gemm_v(sg.BN == 128 ? V_128_6_4 : V_256_4_4, *mx, *mr, *mr, gate_tma ? mlog_f32 : mlog,
                     ctx->at<GemmSched>(s.s_gate), d.H, ctx->num_sms, st));
  }
  ++ctx->launches;
  MARK(1);
  if (fused_gate) {
    k_rank<<<dim3(nchunks, d.GL), 128, 0, st>>>(d, T, ctx->at<int32_t>(s.ids), ctx->at<int32_t>(s.pos),
                                                ctx->at<int32_t>(s.hist));
  } else if (sel) {
    CK(launch_select<false>(d, T, nchunks, st, ctx->at<float>(s.logits), b_router, ctx->at<int32_t>(s.ids),
                            ctx->at<float>(s.gw), ctx->at<int32_t>(s.pos), ctx->at<int32_t>(s.hist), nullptr));
  } else {
    launch_topk<false>(d, T, nchunks, st, ctx->at<float>(s.logits), nullptr, b_router, ctx->at<int32_t>(s.ids),
                       ctx->at<float>(s.gw), ctx->at<int32_t>(s.pos), ctx->at<int32_t>(s.hist), nullptr, nullptr);
  }
  CKL();
  CK(ev_record(ctx, ctx->ev_gate[p], st));
  MARK(2);
  // a3 actual-count all-gather (board kind 0, parity p)
  k_count_scan<<<d.GL, 256, 0, st>>>(d, nchunks, ctx->at<int32_t>(s.hist), ctx->at<int32_t>(s.cbase), sym_of(ctx),
                                     PROBE_BUF_BOARD, p);
  CKL();
  CK(xbarrier(ctx, BAR_COUNTS, st));            // every rank's counts are on every board
  // a5 materialize plan(L) + layout
  if (use_plan) CK(ev_wait(ctx, st, ctx->ev_plan[p]));
  MARK(3);
  LayoutIn li;
  li.board_actual = reinterpret_cast<const int32_t*>(ctx->local_base[PROBE_BUF_BOARD]) + ((p * 2 + 0) * d.G) * d.E;
  li.quota = use_plan ? ctx->at<int32_t>(s.quota[p]) : nullptr;
  li.replicas = use_plan ? ctx->at<int32_t>(s.reps[p]) : nullptr;
  li.bank = p;
  li.nparts = (ctx->ep_emulation && d.GL > 1 && d.GL <= kMaxParts) ? d.GL : 0;
  // CTA pairs pay off when expert groups fill 256-row tiles; decode-sized groups (mean rows per
  // local expert T·k·G/E below 256, e.g. C2: 64) run faster on the 1-CTA kernel (measured:
  // C2 expert GEMMs 1.45 ms on pairs vs 1.15 ms on single CTAs)
  const bool pair = ctx->pair_gemm && static_cast<int64_t>(T) * d.k * d.G >= 256LL * d.E;
  li.tile_m = pair ? 256 : 128;
  const bool g2w = pair && !f32 && ctx->gemm2_512;   // GEMM2 on 256×512 tiles (V_2CTA_512_4_4)
  const bool g1w = pair && !f32 && ctx->gemm1_512;   // GEMM1 (SwiGLU) on 256×512 tiles (256 act columns)
  li.bn2 = g2w ? 512 : 256;
  li.bn1 = g1w ? 512 : 256;
  li.act = ctx->scratch + s.act;
  li.y_local = ctx->local_base[PROBE_BUF_Y];
  li.f32 = f32;
  li.l2hint = ctx->l2hint;
  li.y_wide = ctx->y_wide ? 1 : 0;
  LayoutOut lo;
  lo.split_cum = ctx->at<int32_t>(s.split_cum);
  lo.slot_of = ctx->at<int32_t>(s.slot_of);
  lo.src_off = ctx->at<int32_t>(s.src_off);
  lo.group_rows = ctx->at<int32_t>(s.group_rows);
  lo.replicas_used = ctx->at<int32_t>(s.reps_used);
  lo.s1 = ctx->at<GemmSched>(s.s_g1);
  lo.s2 = ctx->at<GemmSched>(s.s_g2);
  lo.err = err;
  lo.fallbacks = err + kFallbackSlot;
  k_layout<<<1, 512, static_cast<size_t>(d.G) * d.E * d.G * 4, st>>>(d, li, lo);
  CKL();
  MARK(4);
  // a6 dispatch
  const bool dedup = ctx->cfg.dedup_wire != 0;
  const int KQ = d.k < d.G ? d.k : d.G;      // distinct destinations per token, at most
  {
    const int warps = d.GL * T;
    if (dedup) {
      k_dispatch_dedup<<<(warps + 7) / 8, 256, 0, st>>>(d, T, static_cast<const uint8_t*>(x), row_bytes,
                                                       ctx->at<int32_t>(s.ids), ctx->at<int32_t>(s.pos),
                                                       ctx->at<int32_t>(s.cbase), lo.split_cum, lo.slot_of,
                                                       lo.src_off, ctx->at<int32_t>(s.route), ctx->at<float>(s.gw),
                                                       sym_of(ctx), PROBE_BUF_RECV, PROBE_BUF_META, KQ, err,
                                                       predisp ? ctx->at<int32_t>(s.pids[p]) : nullptr,
                                                       err + kHitSlot);
    } else {
      k_dispatch<<<(warps + 7) / 8, 256, 0, st>>>(d, T, static_cast<const uint8_t*>(x), row_bytes,
                                                  ctx->at<int32_t>(s.ids),
                                                  ctx->at<int32_t>(s.pos), ctx->at<int32_t>(s.cbase),
                                                  lo.split_cum, lo.slot_of, lo.src_off, ctx->at<int32_t>(s.route),
                                                  sym_of(ctx), PROBE_BUF_RECV, err);
    }
    CKL();
  }
  CK(ev_record(ctx, ctx->ev_disp[p], st));
  if (predisp) CK(ev_wait(ctx, st, ctx->ev_pd_done));  // pre-dispatched rows complete before the barrier
  CK(xbarrier(ctx, BAR_DISPATCH, st));                // every peer's rows have landed in our receive buffers
  MARK(5);
  if (dedup) {
    // receiver: expand each (token, dest) wire row into the pair's other slot rows (local HBM)
    k_expand<<<ctx->num_sms * 4, 256, 0, st>>>(d, lo.group_rows, sym_of(ctx), PROBE_BUF_META, PROBE_BUF_RECV,
                                               row_bytes, T, KQ, PROBE_BUF_PRE, ctx->cfg.max_tokens);
    CKL();
  }
  MARK(6);
  // a9 phase lock: the expert GEMMs need this layer's replica slots
  if (use_plan) CK(ev_wait(ctx, st, ctx->ev_slots[p]));
  MARK(7);
  CK(ev_record(ctx, ctx->ev_gemm[p], st));
  // a7 grouped SwiGLU expert FFN (tcgen05): act = SiLU(X W_gᵀ) ⊙ X W_uᵀ ; Y = act W_dᵀ
  const int vexp = pair ? V_2CTA_256_6_4 : V_256_4_4_EXP;
  // R26: the measured hiding window starts with the expert GEMMs
  k_window_stamp<<<1, 1, 0, st>>>(d, ctx->at<int64_t>(s.win_t0), 0, sym_of(ctx), PROBE_BUF_BOARD, lo.group_rows,
                                  ctx->cfg.n_sat);
  CKL();
  if (f32) {
    CK(launch_sgemm(ctx, lo.s1, ctx->local_base[PROBE_BUF_RECV], w13, ctx->local_base[PROBE_BUF_REP_W13], d.H, st));
  } else {
    CK(launch_gemm_v(g1w ? V_2CTA_512_4_4 : vexp, ctx->map_recv, *m13, ctx->map_rw13, ctx->map_act_out, lo.s1, d.H,
                     ctx->num_sms, st));
  }
  ++ctx->launches;
  if (ctx->dbg_gap_us > 0) k_spin<<<1, 1, 0, st>>>(ctx->dbg_gap_us * 1000ll);
  MARK(8);
  if (f32) {
    CK(launch_sgemm(ctx, lo.s2, ctx->scratch + s.act, w2, ctx->local_base[PROBE_BUF_REP_W2], d.F, st));
  } else {
    // double-buffered wide stores need the ≤ 384-group table of the NB2 instance (C1: 8 × 19 groups,
    // C3: 8 × 35)
    const int v2 = !g2w ? vexp : (ctx->g2_nb2 && d.GL * (d.EL + kMaxRb) <= 384 ? V_2CTA_512_4_4_NB2 : V_2CTA_512_4_4);
    CK(launch_gemm_v(v2, ctx->map_act, *m2, ctx->map_rw2, ctx->map_y, lo.s2, d.F, ctx->num_sms, st));
    if (ctx->dbg_gemm2_repeat && li.nparts == 0) {   // same result again, after a GEMM2 instead of a GEMM1
      CK(cudaMemsetAsync(&lo.s2->counter, 0, sizeof(int32_t), st));
      CK(launch_gemm_v(v2, ctx->map_act, *m2, ctx->map_rw2, ctx->map_y, lo.s2, d.F, ctx->num_sms, st));
    }
  }
  ++ctx->launches;
  k_window_stamp<<<1, 64, 0, st>>>(d, ctx->at<int64_t>(s.win_t0), 1, sym_of(ctx), PROBE_BUF_BOARD, lo.group_rows,
                                  ctx->cfg.n_sat);
  CKL();
  if (!dedup) CK(xbarrier(ctx, BAR_Y, st));     // every expert rank's Y rows are complete (the combine pulls)
  MARK(9);
  // a8 combine (raises the prefetch suspend flag, R27)
  if (dedup) {
    // expert side: one fp32 partial per (token, dest) over its co-located slots → the source's COMB (R25)
#define PARTIAL(YF, KC)                                                                                      \
  k_combine_partial<YF, KC><<<ctx->num_sms * 4, 256, 0, st>>>(d, T, lo.group_rows, sym_of(ctx), PROBE_BUF_META, \
                                                              PROBE_BUF_Y, PROBE_BUF_COMB, KQ, suspend, layer)
    if (f32 && d.k <= 8) PARTIAL(true, 8);
    else if (f32) PARTIAL(true, kMaxK);
    else if (d.k <= 8) PARTIAL(false, 8);
    else PARTIAL(false, kMaxK);
#undef PARTIAL
    CKL();
    CK(xbarrier(ctx, BAR_Y, st));               // every expert rank's partials have landed on their sources
  } else if (f32 && out_fp32)
    k_combine<true, true><<<d.GL * T, 128, 0, st>>>(d, T, ctx->at<float>(s.gw), ctx->at<int32_t>(s.route),
                                                    sym_of(ctx), PROBE_BUF_Y, out, suspend, layer);
  else if (f32)
    k_combine<false, true><<<d.GL * T, 128, 0, st>>>(d, T, ctx->at<float>(s.gw), ctx->at<int32_t>(s.route),
                                                     sym_of(ctx), PROBE_BUF_Y, out, suspend, layer);
  else {
#define COMBINE(OF, KC)                                                                                   \
  k_combine<OF, false, KC><<<d.GL * T, 128, 0, st>>>(d, T, ctx->at<float>(s.gw), ctx->at<int32_t>(s.route), \
                                                     sym_of(ctx), PROBE_BUF_Y, out, suspend, layer)
    if (out_fp32 && d.k <= 8) COMBINE(true, 8);
    else if (out_fp32) COMBINE(true, kMaxK);
    else if (d.k <= 8) COMBINE(false, 8);
    else COMBINE(false, kMaxK);
#undef COMBINE
  }
  CKL();
  MARK(10);
  if (dedup) {
    // source side: Σ of the token's partials in ascending destination order (R25)
    const int* rt_ = ctx->at<int32_t>(s.route);
    if (f32 && out_fp32) k_combine_reduce<true, true><<<d.GL * T, 128, 0, st>>>(d, T, rt_, sym_of(ctx), PROBE_BUF_COMB, KQ, out);
    else if (f32) k_combine_reduce<false, true><<<d.GL * T, 128, 0, st>>>(d, T, rt_, sym_of(ctx), PROBE_BUF_COMB, KQ, out);
    else if (out_fp32) k_combine_reduce<true, false><<<d.GL * T, 128, 0, st>>>(d, T, rt_, sym_of(ctx), PROBE_BUF_COMB, KQ, out);
    else k_combine_reduce<false, false><<<d.GL * T, 128, 0, st>>>(d, T, rt_, sym_of(ctx), PROBE_BUF_COMB, KQ, out);
    CKL();
  }
  CK(ev_record(ctx, ctx->ev_comb[p], st));
  MARK(11);
  if (prof) ++ctx->prof_n;
#undef MARK
  if (topk_ids) CK(cudaMemcpyAsync(topk_ids, ctx->at<int32_t>(s.ids), GL * T * d.k * 4, cudaMemcpyDeviceToDevice, st));
  if (topk_w) CK(cudaMemcpyAsync(topk_w, ctx->at<float>(s.gw), GL * T * d.k * 4, cudaMemcpyDeviceToDevice, st));
  ctx->fwd_layer = layer;
  ctx->last_fwd_parity = p;
  ctx->last_T = T;
  return PROBE_OK;
}

probe_status probe_predict(probe_ctx ctx, int32_t next_layer, const void* x, int32_t T, const void* w_router_next,
                           const float* b_router_next, const void* w_res1, const void* w_res2, int32_t* pred_counts,
                           float* pred_logits, void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  if (!x || !w_router_next) return fail(ctx, PROBE_EINVAL, "probe_predict: null pointer");
  if ((w_res1 == nullptr) != (w_res2 == nullptr)) return fail(ctx, PROBE_EINVAL, "w_res1 and w_res2 must both be given or both NULL");
  if (w_res1 && ctx->cfg.res_hidden <= 0) return fail(ctx, PROBE_ESHAPE, "residual given but res_hidden == 0");
  if (T < 1 || T > ctx->cfg.max_tokens) return fail(ctx, PROBE_ECAPACITY, "T=%d outside [1, max_tokens]", T);
  if (next_layer < 1) return fail(ctx, PROBE_EINVAL, "next_layer %d < 1 (layer 0 is not predicted, R29)", next_layer);
  Dims d = ctx->d;
  d.T = T;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->aux;
  const int pp = next_layer & 1, prev = (next_layer - 1) & 1;
  if (ctx->fwd_layer == next_layer - 1)
    CK(ev_wait(ctx, st, ctx->aux_start ? ctx->ev_disp[prev] : ctx->ev_gate[prev]));
  const uint64_t GL = d.GL, H = d.H, E = d.E, h = d.h;
  const Scratch& s = ctx->sl;
  const bool f32 = ctx->f32();
  const CUtensorMap* mx = f32 ? nullptr : ctx->maps.get(x, GL * T, H, 128);
  if (!f32 && !mx) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
  const int nchunks = (T + kChunk - 1) / kChunk;
  CK(cudaMemsetAsync(ctx->at<int32_t>(s.pred_local), 0, GL * E * 4, st));
  // The product path (K-concatenated GEMM + k_select) also serves pred_logits requests: the
  // select kernel writes l̂ = prior + residual + b as it ranks it, so the logits a caller
  // inspects are the ones that produced n̂ (only the debug/unfused path and k > 8 differ).
  const bool fused = d.k <= kTopkMax && d.E <= 256 && !ctx->unfused;
  // epilogue top-k keeps neither logits nor per-token sets (NEXT-4 pre-dispatch needs the sets)
  const bool epi_topk = ctx->fused_epi_topk && !pred_logits && !ctx->cfg.predispatch;
  int32_t* pids = ctx->cfg.predispatch ? ctx->at<int32_t>(s.pids[pp]) : nullptr;
  // stage 1 (prior W_{L+1}·x and a = bf16(SiLU(Ŵ1 x))) already computed by the fused gate GEMM
  // of probe_moe_forward(next_layer-1) for exactly these operands?
  const auto& gd = ctx->gp_done[pp];
  const bool gp = ctx->cfg.fuse_gate_predictor && fused && !f32 && gd.layer == next_layer && gd.x == x &&
                  gd.T == T && gd.wn == w_router_next && gd.w1 == w_res1;
  if (gp) {
    // stage 2: residual Ŵ2·a (1-CTA kernel, K = h, fp32 by TMA tensor stores), then the top-k
    // select forms l̂ = prior + residual + b and writes n̂ (Eq. (P), R9)
    const float* prior = ctx->at<float>(s.gprior[pp]);
    const float* resid = nullptr;
    if (w_res1) {
      const int BN = d.E <= 128 ? 128 : 256;
      const CUtensorMap* ma = ctx->maps.get(ctx->scratch + s.gact[pp], GL * T, h, 128);
      const CUtensorMap* m2 = ctx->maps.get(w_res2, E, h, BN / 2);
      if (!ma || !m2) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
      CUtensorMap mres;
      if (!make_map_f32_out(&mres, ctx->scratch + s.pres, GL * T, E)) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
      SmallGroups s2{};
      s2.BN = BN;
      s2.n = 1;
      s2.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.pres));
      s2.g[0].tma_out = 1;                      // E % 32 == 0 (fuse_gate_predictor requires it)
      k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p2), s2);
      CKL();
      CK(launch_gemm_v(BN == 128 ? V_128_6_4 : V_256_4_4, *ma, *m2, *m2, mres, ctx->at<GemmSched>(s.s_p2), d.h,
                       ctx->aux_sms, st));
      ++ctx->launches;
      resid = ctx->at<float>(s.pres);
    }
    CK(launch_select<true>(d, T, nchunks, st, prior, b_router_next, nullptr, nullptr, nullptr, nullptr,
                           ctx->at<int32_t>(s.pred_local), pred_logits, pids, resid));
    ++ctx->launches;
  } else if (f32) {
    // fp32 parity path: prior x·W_{L+1}ᵀ and z = x·Ŵ1ᵀ → a = bf16(SiLU(z)) (R8) in one grouped
    // SIMT launch, residual a·Ŵ2ᵀ, then the warp top-k sums prior + b + residual (Eq. (P))
    SmallGroups sg{};
    sg.BN = 128;
    sg.n = w_res1 ? 2 : 1;
    sg.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.pprior));
    if (w_res1) sg.g[1] = mk_group(0, static_cast<int>(GL * T), 0, 1, EPI_SILU_BF16, d.h, d.h, ctx->scratch + s.pact);
    k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p1), sg);
    CKL();
    CK(launch_sgemm(ctx, ctx->at<GemmSched>(s.s_p1), x, w_router_next, w_res1 ? w_res1 : w_router_next, d.H, st));
    ++ctx->launches;
    if (w_res1) {
      SmallGroups s2{};
      s2.BN = 128;
      s2.n = 1;
      s2.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.pres));
      k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p2), s2);
      CKL();
      CK(launch_sgemm(ctx, ctx->at<GemmSched>(s.s_p2), ctx->scratch + s.pact, w_res2, w_res2, d.h, st));
      ++ctx->launches;
    }
    launch_topk<true>(d, T, nchunks, st, ctx->at<float>(s.pprior), w_res1 ? ctx->at<float>(s.pres) : nullptr,
                      b_router_next, nullptr, nullptr, nullptr, nullptr, ctx->at<int32_t>(s.pred_local), pred_logits);
    CKL();
  } else if (fused) {
    // (1) a = bf16(SiLU(Ŵ1 x))  [GL·T, h]   (2) l̂ = [x | a]·[W_{L+1} | Ŵ2]ᵀ (+b) with the
    // top-k and the per-rank count n̂ fused in the epilogue (one TMEM accumulator for prior
    // + residual; Eq. (P), R8, R9).
    const int BN = d.E <= 128 ? 128 : 256;
    const CUtensorMap* mw = ctx->maps.get(w_router_next, E, H, BN / 2);
    const CUtensorMap* ma = nullptr;
    const CUtensorMap* m2 = nullptr;
    if (w_res1) {
      // z = x Ŵ1ᵀ (N = h): on CTA pairs (256×256 tiles, tcgen05 cta_group::2) when h fills a
      // 256-column tile — it is 75% of the predictor's FLOPs (C1: 137 of 180 GFLOP), and the
      // 1-CTA <128,6,4> kernel ran it at 56% of its SMs' peak beside the dispatch
      const bool pair1 = ctx->pred_pair && d.h >= 256 && static_cast<int64_t>(GL) * T >= 256;
      const CUtensorMap* m1 = ctx->maps.get(w_res1, h, H, pair1 ? 128 : 64);
      ma = ctx->maps.get(ctx->scratch + s.pact, GL * T, h, 128);
      m2 = ctx->maps.get(w_res2, E, h, BN / 2);
      if (!m1 || !ma || !m2) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
      SmallGroups s1{};
      s1.BN = pair1 ? 256 : 128;
      s1.TM = pair1 ? 256 : 128;
      s1.n = 1;
      s1.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_SILU_BF16, d.h, d.h, ctx->scratch + s.pact);
      // a = bf16(SiLU(z)) written by TMA tensor stores (per-lane stores halved this GEMM's rate)
      CUtensorMap mact;
      const bool tma_act = d.h % 32 == 0 && make_map_bf16_out(&mact, ctx->scratch + s.pact, GL * T, h);
      s1.g[0].tma_out = tma_act ? 1 : 0;
      k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p1), s1);
      CKL();
      const int v1 = pair1 ? V_2CTA_256_6_4 : (ctx->pred_maxreg ? V_128_6_4_R192 : V_128_6_4);
      CK(launch_gemm_v(v1, *mx, *m1, *m1, tma_act ? mact : *mx, ctx->at<GemmSched>(s.s_p1), d.H, ctx->aux_sms, st));
      ++ctx->launches;
    }
    if (!mw) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
    // the K-concatenated prior + residual GEMM on CTA pairs as well (not with the epilogue top-k)
    const bool pair2 = ctx->pred_pair && !epi_topk && static_cast<int64_t>(GL) * T >= 256;
    SmallGroups s2{};
    s2.BN = BN;
    s2.TM = pair2 ? 256 : 128;
    s2.n = 1;
    if (epi_topk) {
      s2.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_TOPK_COUNT, d.E, d.E, nullptr);
      s2.g[0].topk = d.k;
      s2.g[0].rows_per_rank = T;
      s2.g[0].aux = ctx->at<int32_t>(s.pred_local);
      s2.g[0].bias = b_router_next;
    } else {
      s2.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.pprior));
    }
    CUtensorMap mpr;
    const bool pr_tma = !epi_topk && d.E % 32 == 0 && make_map_f32_out(&mpr, ctx->at<float>(s.pprior), GL * T, E);
    if (pr_tma) s2.g[0].tma_out = 1;
    k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p2), s2);
    CKL();
    const int v2 = pair2 ? (BN == 128 ? V_2CTA_128_8_4 : V_2CTA_256_6_4)
                         : (BN == 128 ? (ctx->pred_maxreg ? V_128_6_4_R192 : V_128_6_4) : V_256_4_4);
    CK(launch_gemm_v(v2, *mx, *mw, w_res1 ? *m2 : *mw, pr_tma ? mpr : *mx, ctx->at<GemmSched>(s.s_p2), d.H,
                     ctx->aux_sms, st, w_res1 ? ma : nullptr, w_res1 ? d.h : 0));
    ++ctx->launches;
    if (!epi_topk) {
      CK(launch_select<true>(d, T, nchunks, st, ctx->at<float>(s.pprior), b_router_next, nullptr, nullptr, nullptr,
                             nullptr, ctx->at<int32_t>(s.pred_local), pred_logits, pids));
      ++ctx->launches;
    }
  } else {
    // unfused (debug / k > 8): prior + SiLU activation, residual GEMM, warp top-k; writes logits
    const CUtensorMap* mw = ctx->maps.get(w_router_next, E, H, 64);
    const CUtensorMap* m1 = w_res1 ? ctx->maps.get(w_res1, h, H, 64) : mw;
    if (!mw || !m1) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
    SmallGroups sg{};
    sg.BN = 128;
    sg.n = w_res1 ? 2 : 1;
    sg.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.pprior));
    if (w_res1) sg.g[1] = mk_group(0, static_cast<int>(GL * T), 0, 1, EPI_SILU_BF16, d.h, d.h, ctx->scratch + s.pact);
    k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p1), sg);
    CKL();
    CK(launch_gemm_v(V_128_6_4, *mx, *mw, *m1, *mx, ctx->at<GemmSched>(s.s_p1), d.H, ctx->aux_sms, st));
    ++ctx->launches;
    if (w_res1) {
      const CUtensorMap* ma = ctx->maps.get(ctx->scratch + s.pact, GL * T, h, 128);
      const CUtensorMap* m2 = ctx->maps.get(w_res2, E, h, 64);
      if (!ma || !m2) return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
      SmallGroups s2{};
      s2.BN = 128;
      s2.n = 1;
      s2.g[0] = mk_group(0, static_cast<int>(GL * T), 0, 0, EPI_F32, d.E, d.E, ctx->at<float>(s.pres));
      k_write_sched<<<1, 32, 0, st>>>(ctx->at<GemmSched>(s.s_p2), s2);
      CKL();
      CK(launch_gemm_v(V_128_6_4, *ma, *m2, *m2, *ma, ctx->at<GemmSched>(s.s_p2), d.h, ctx->aux_sms, st));
      ++ctx->launches;
    }
    launch_topk<true>(d, T, nchunks, st, ctx->at<float>(s.pprior), w_res1 ? ctx->at<float>(s.pres) : nullptr,
                      b_router_next, nullptr, nullptr, nullptr, nullptr, ctx->at<int32_t>(s.pred_local), pred_logits);
    CKL();
  }
  k_pred_publish<<<d.GL, 256, 0, st>>>(d, ctx->at<int32_t>(s.pred_local), sym_of(ctx), PROBE_BUF_BOARD, pp);
  CKL();
  CK(xbarrier(ctx, BAR_PRED, st));              // n̂ of every rank on every board
  if (pred_counts) {
    const int32_t* board = reinterpret_cast<const int32_t*>(ctx->local_base[PROBE_BUF_BOARD]) + ((pp * 2 + 1) * d.G) * d.E;
    CK(cudaMemcpyAsync(pred_counts, board, static_cast<size_t>(d.G) * d.E * 4, cudaMemcpyDeviceToDevice, st));
  }
  CK(ev_record(ctx, ctx->ev_pred[pp], st));
  ctx->pred_layer[pp] = next_layer;
  ctx->pred_T[pp] = (pids && fused && !f32) ? T : 0;   // per-token sets exist only on the select path
  return PROBE_OK;
}

probe_status probe_predict_prepare(probe_ctx ctx, int32_t next_layer, const void* w_router_next,
                                   const void* w_res1) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  if (!ctx->cfg.fuse_gate_predictor)
    return fail(ctx, PROBE_ESTATE, "probe_predict_prepare: probe_config.fuse_gate_predictor is 0");
  if (!w_router_next) return fail(ctx, PROBE_EINVAL, "probe_predict_prepare: null w_router_next");
  if (w_res1 && ctx->cfg.res_hidden <= 0) return fail(ctx, PROBE_ESHAPE, "residual given but res_hidden == 0");
  if (next_layer < 1) return fail(ctx, PROBE_EINVAL, "next_layer %d < 1 (layer 0 is not predicted, R29)", next_layer);
  ctx->gp_next = next_layer;
  ctx->gp_wn = w_router_next;
  ctx->gp_w1 = w_res1;
  return PROBE_OK;
}

probe_status probe_plan(probe_ctx ctx, int32_t next_layer, const int32_t* pred_counts, const int64_t* window_ns,
                        int32_t* replicas, int32_t* quota, int64_t* plan_stats, void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  if (!window_ns) return fail(ctx, PROBE_EINVAL, "probe_plan: window_ns is required");
  if (next_layer < 0) return fail(ctx, PROBE_EINVAL, "next_layer < 0");
  const int pp = next_layer & 1;
  if (!pred_counts && ctx->pred_layer[pp] != next_layer)
    return fail(ctx, PROBE_ESTATE, "probe_plan(%d): no probe_predict(%d) and no explicit pred_counts", next_layer, next_layer);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->aux;
  const Dims& d = ctx->d;
  const Scratch& s = ctx->sl;
  if (!pred_counts) CK(ev_wait(ctx, st, ctx->ev_pred[pp]));
  const int32_t* nh = pred_counts ? pred_counts
                                  : reinterpret_cast<const int32_t*>(ctx->local_base[PROBE_BUF_BOARD]) + ((pp * 2 + 1) * d.G) * d.E;
  PlanParams pr{ctx->cfg.alpha_ps, ctx->cfg.beta_ps, ctx->cfg.bw_bytes_per_us, ctx->cfg.expert_bytes,
                ctx->cfg.n_sat, ctx->cfg.kmax, ctx->cfg.replica_budget};
  const size_t smem = static_cast<size_t>(d.G) * d.E * d.G * 4;    // quota bytes
  k_plan<<<1, 64, 0, st>>>(d, pr, nh, window_ns, ctx->at<int32_t>(s.quota[pp]), ctx->at<int32_t>(s.reps[pp]),
                            ctx->at<int64_t>(s.stats[pp]), ctx->at<int32_t>(s.pfctr[pp]));
  CKL();
  if (replicas) CK(cudaMemcpyAsync(replicas, ctx->at<int32_t>(s.reps[pp]), d.G * kMaxRb * 4, cudaMemcpyDeviceToDevice, st));
  if (quota) CK(cudaMemcpyAsync(quota, ctx->at<int32_t>(s.quota[pp]), smem, cudaMemcpyDeviceToDevice, st));
  if (plan_stats) CK(cudaMemcpyAsync(plan_stats, ctx->at<int64_t>(s.stats[pp]), 64, cudaMemcpyDeviceToDevice, st));
  CK(ev_record(ctx, ctx->ev_plan[pp], st));
  ctx->plan_layer[pp] = next_layer;
  return PROBE_OK;
}

probe_status probe_prefetch(probe_ctx ctx, int32_t next_layer, const void* w13_next, const void* w2_next, int32_t phase,
                            void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  const int pp = next_layer & 1, prev = (next_layer - 1) & 1;
  if (phase == 1) {
    if (ctx->pf_layer[pp] != next_layer) return fail(ctx, PROBE_ESTATE, "prefetch WAIT(%d) before START", next_layer);
    CK(ev_wait(ctx, static_cast<cudaStream_t>(stream), ctx->ev_slots[pp]));
    return PROBE_OK;
  }
  if (phase != 0) return fail(ctx, PROBE_EINVAL, "phase must be 0 (START) or 1 (WAIT)");
  if (!w13_next || !w2_next) return fail(ctx, PROBE_EINVAL, "probe_prefetch: null weights");
  if (ctx->plan_layer[pp] != next_layer) return fail(ctx, PROBE_ESTATE, "prefetch START(%d) before probe_plan(%d)", next_layer, next_layer);
  const Dims& d = ctx->d;
  const Scratch& s = ctx->sl;
  cudaStream_t st = ctx->pf;
  CK(ev_wait(ctx, st, ctx->ev_plan[pp]));
  int32_t* flags = ctx->at<int32_t>(s.flags);
  const bool inflight = ctx->fwd_layer == next_layer - 1;
  const int grid = 16;  // part 2 (after the combine): "controlled SM occupancy"
  if (inflight) {
    // part 1 beside the expert GEMMs: one 128-thread CTA per SM fits in the registers the
    // register-capped expert GEMM CTAs leave free (kExpertMaxReg × 256 + kPrefetchPart1Reg × 128 ≤ 62 K)
    CK(ev_wait(ctx, st, ctx->ev_gemm[prev]));
    k_prefetch<kPrefetchPart1Reg, 8><<<ctx->num_sms, 128, 0, st>>>(d, ctx->at<int32_t>(s.reps[pp]), pp, static_cast<const uint8_t*>(w13_next),
                                     static_cast<const uint8_t*>(w2_next), sym_of(ctx), PROBE_BUF_REP_W13,
                                     PROBE_BUF_REP_W2, ctx->at<int32_t>(s.pfctr[pp]), flags + 1, next_layer,
                                     flags + 2, static_cast<int>(esz(ctx->cfg)));
    CKL();
    CK(ev_wait(ctx, st, ctx->ev_comb[prev]));
  }
  k_prefetch<><<<grid, 512, 0, st>>>(d, ctx->at<int32_t>(s.reps[pp]), pp, static_cast<const uint8_t*>(w13_next),
                                   static_cast<const uint8_t*>(w2_next), sym_of(ctx), PROBE_BUF_REP_W13,
                                   PROBE_BUF_REP_W2, ctx->at<int32_t>(s.pfctr[pp]), flags + 1, -1, flags + 3,
                                   static_cast<int>(esz(ctx->cfg)));
  CKL();
  CK(xbarrier(ctx, BAR_PREFETCH, st));          // every sender finished pushing into our slots
  CK(ev_record(ctx, ctx->ev_slots[pp], st));
  ctx->pf_layer[pp] = next_layer;
  return PROBE_OK;
}

probe_status probe_debug_prefetch(probe_ctx ctx, int32_t* out, void* stream) {
  if (!ctx || !out) return fail(ctx, PROBE_EINVAL, "probe_debug_prefetch: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ev, ctx->pf));
  CK(cudaStreamWaitEvent(st, ev, 0));
  CK(cudaEventDestroy(ev));
  CK(cudaMemcpyAsync(out, ctx->at<int32_t>(ctx->sl.flags) + 2, 8, cudaMemcpyDeviceToDevice, st));
  return PROBE_OK;
}

probe_status probe_window(probe_ctx ctx, int64_t attention_ns, int64_t fallback_ns, int64_t* window_ns,
                          void* stream) {
  if (!ctx || !window_ns) return fail(ctx, PROBE_EINVAL, "probe_window: null argument");
  if (attention_ns < 0 || fallback_ns < 0) return fail(ctx, PROBE_EINVAL, "probe_window: negative time");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->aux;
  k_window_read<<<1, 64, 0, st>>>(ctx->d, ctx->local_base[PROBE_BUF_BOARD], attention_ns, fallback_ns, window_ns);
  CKL();
  return PROBE_OK;
}

probe_status probe_debug_flags(probe_ctx ctx, int32_t* out, void* stream) {
  if (!ctx || !out) return fail(ctx, PROBE_EINVAL, "probe_debug_flags: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ev, ctx->pf));
  CK(cudaStreamWaitEvent(st, ev, 0));
  CK(cudaEventRecord(ev, ctx->aux));
  CK(cudaStreamWaitEvent(st, ev, 0));
  CK(cudaEventDestroy(ev));
  CK(cudaMemcpyAsync(out, ctx->at<int32_t>(ctx->sl.flags), 8 * 4, cudaMemcpyDeviceToDevice, st));
  return PROBE_OK;
}

probe_status probe_debug_layout(probe_ctx ctx, int32_t* counts, int32_t* split, int32_t* route, int32_t* group_rows,
                                int32_t* replicas_used, void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims& d = ctx->d;
  const Scratch& s = ctx->sl;
  const int p = ctx->last_fwd_parity;
  if (counts) {
    const int32_t* b = reinterpret_cast<const int32_t*>(ctx->local_base[PROBE_BUF_BOARD]) + ((p * 2 + 0) * d.G) * d.E;
    CK(cudaMemcpyAsync(counts, b, static_cast<size_t>(d.G) * d.E * 4, cudaMemcpyDeviceToDevice, st));
  }
  if (split) CK(cudaMemcpyAsync(split, ctx->at<int32_t>(s.split_cum), static_cast<size_t>(d.G) * d.E * d.G * 4, cudaMemcpyDeviceToDevice, st));
  if (route) CK(cudaMemcpyAsync(route, ctx->at<int32_t>(s.route), static_cast<size_t>(d.GL) * ctx->last_T * d.k * 8, cudaMemcpyDeviceToDevice, st));
  if (group_rows)
    CK(cudaMemcpyAsync(group_rows, ctx->at<int32_t>(s.group_rows) + d.R0 * (d.EL + kMaxRb),
                       static_cast<size_t>(d.GL) * (d.EL + kMaxRb) * 4, cudaMemcpyDeviceToDevice, st));
  if (replicas_used) CK(cudaMemcpyAsync(replicas_used, ctx->at<int32_t>(s.reps_used), d.G * kMaxRb * 4, cudaMemcpyDeviceToDevice, st));
  return PROBE_OK;
}

probe_status probe_test_gemm(const void* A, int64_t a_rows, const void* B, int64_t b_rows, int32_t K, int32_t N,
                             const int32_t* groups, int32_t num_groups, int32_t mode, void* C, void* stream) {
  return probe_bench_gemm(A, a_rows, B, b_rows, K, N, groups, num_groups, mode, -1, 1, nullptr, C, stream);
}

probe_status probe_bench_gemm(const void* A, int64_t a_rows, const void* B, int64_t b_rows, int32_t K, int32_t N,
                              const int32_t* groups, int32_t num_groups, int32_t mode, int32_t variant, int32_t reps,
                              float* ms_out, void* C, void* stream) {
  probe_ctx ctx = nullptr;
  if (!A || !B || !groups || !C || num_groups < 1 || num_groups > kMaxGroups || K < 1 || N < 8 || N % 8 ||
      reps < 1 || mode < 0 || mode > 7)
    return fail(nullptr, PROBE_EINVAL, "probe_test_gemm: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant < 0) variant = mode == 1 || mode == 2 ? V_256_4_4 : V_128_6_4;
  if (!variant_ok(variant)) return fail(nullptr, PROBE_EINVAL, "variant %d not available", variant);
  const int TM = variant_tm(variant);
  const int BN = variant_bn(variant);
  const int emode = mode == 1 ? EPI_SWIGLU
                    : mode == 3 ? EPI_SILU_BF16
                    : mode == 4 ? EPI_NONE
                    : mode == 5 ? EPI_TOPK
                    : mode == 6 ? EPI_TOPK_COUNT
                    : mode == 7 ? EPI_F16 : EPI_F32;
  void* topk_aux = nullptr;
  if (emode == EPI_TOPK || emode == EPI_TOPK_COUNT) {
    if (N > 256) return fail(nullptr, PROBE_EINVAL, "top-k modes need N <= 256");
    CK(cudaMalloc(&topk_aux, static_cast<size_t>(a_rows) * 8 * 4 + static_cast<size_t>(N) * 4 * 64));
    CK(cudaMemset(topk_aux, 0, static_cast<size_t>(a_rows) * 8 * 4 + static_cast<size_t>(N) * 4 * 64));
  }
  const int n_out = mode == 1 ? N / 2 : N;
  std::vector<uint8_t> host(sizeof(GemmSched), 0);
  GemmSched* hs = reinterpret_cast<GemmSched*>(host.data());
  hs->num_groups = num_groups;
  if (const char* h = getenv("PROBE_L2HINT")) hs->l2hint = static_cast<int>(strtol(h, nullptr, 0)) & 7;
  unsigned long long* dstats = nullptr;
  if (getenv("PROBE_GEMM_STATS")) {
    CK(cudaMalloc(&dstats, 8 * sizeof(unsigned long long)));
    CK(cudaMemset(dstats, 0, 8 * sizeof(unsigned long long)));
    hs->stats = dstats;
  }
  const size_t esz = emode == EPI_SWIGLU || emode == EPI_SILU_BF16 || emode == EPI_F16 ? 2 : 4;
  // PROBE_Y_WIDE=0/1: fp16 outputs by 32- or 64-column TMA stores (A/B of epi_chunk64_f16)
  const bool y_wide = n_out % 64 == 0 && !(getenv("PROBE_Y_WIDE") && getenv("PROBE_Y_WIDE")[0] == '0');
  int acc = 0;
  int64_t c_rows = 1;
  for (int i = 0; i < num_groups; ++i) {
    const int* g = groups + 4 * i;
    hs->g[i] = mk_group(g[0], g[1], g[2], 0, emode, n_out, n_out, static_cast<uint8_t*>(C) + static_cast<size_t>(g[3]) * n_out * esz);
    hs->g[i].out_row = g[3];
    hs->g[i].tma_out =
        (emode == EPI_F32 || emode == EPI_F16 || emode == EPI_SWIGLU || emode == EPI_SILU_BF16) && n_out % 32 == 0 &&
                !getenv("PROBE_NO_TMA_OUT") ? 1 : 0;      // analysis: coalesced st.global epilogue instead
    if (y_wide && emode == EPI_F16 && hs->g[i].tma_out) hs->g[i].tma_out = 2;
    if (topk_aux) {   // test hook: k = 8; TOPK writes ids to C, weights to aux; COUNT: counts [64][N]
      hs->g[i].topk = 8;
      hs->g[i].rows_per_rank = static_cast<int>((a_rows + 63) / 64);
      hs->g[i].aux = topk_aux;
      hs->g[i].out = static_cast<uint8_t*>(C) + static_cast<size_t>(g[3]) * 8 * 4;
    }
    c_rows = std::max<int64_t>(c_rows, static_cast<int64_t>(g[3]) + g[1]);
    hs->g[i].tile_start = acc;
    acc += gemm_ntiles(hs->g[i], BN, TM);
  }
  hs->total_tiles = acc;
  hs->tile_m = TM;
  CUtensorMap ma, mb, mc;
  if (!make_map(&ma, A, a_rows, K, 128) || !make_map(&mb, B, b_rows, K, BN >= 512 ? 128 : BN / 2))
    return fail(nullptr, PROBE_ECUDA, "tensor map encode failed");
  if (emode == EPI_F32 && n_out % 32 == 0) {
    if (!make_map_f32_out(&mc, C, c_rows, n_out)) return fail(nullptr, PROBE_ECUDA, "tensor map encode failed");
  } else if (emode == EPI_F16 && n_out % 32 == 0) {
    if (!make_map_f16_out(&mc, C, c_rows, n_out, y_wide)) return fail(nullptr, PROBE_ECUDA, "tensor map encode failed");
  } else if ((emode == EPI_SWIGLU || emode == EPI_SILU_BF16) && n_out % 32 == 0) {
    if (!make_map_bf16_out(&mc, C, c_rows, n_out)) return fail(nullptr, PROBE_ECUDA, "tensor map encode failed");
  } else {
    mc = ma;
  }
  GemmSched* ds = nullptr;
  CK(cudaMalloc(&ds, sizeof(GemmSched)));
  CK(cudaMemcpy(ds, hs, sizeof(GemmSched), cudaMemcpyHostToDevice));
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // the dynamic tile counter is reset before every launch (the forward path resets it in
  // the kernel that writes the schedule)
  cudaError_t e = cudaMemsetAsync(&ds->counter, 0, sizeof(int32_t), st);
  if (e == cudaSuccess) e = launch_gemm_v(variant, ma, mb, mb, mc, ds, K, sms, st);   // warm-up / single run
  if (e == cudaSuccess && reps > 1) {
    e = cudaEventRecord(e0, st);
    for (int r = 0; r < reps && e == cudaSuccess; ++r) {
      e = cudaMemsetAsync(&ds->counter, 0, sizeof(int32_t), st);
      if (e == cudaSuccess) e = launch_gemm_v(variant, ma, mb, mb, mc, ds, K, sms, st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(e1, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && reps > 1 && ms_out) {
    float t = 0.f;
    e = cudaEventElapsedTime(&t, e0, e1);
    *ms_out = t / reps;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(ds);
  if (topk_aux) cudaFree(topk_aux);
  if (dstats) {
    unsigned long long h[8];
    if (cudaMemcpy(h, dstats, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess)
      fprintf(stderr, "[gemm stats] variant %d reps %d: prod_wait_empty %.3g  mma_wait_full %.3g  mma_wait_tempty %.3g  "
                      "epi_wait_tfull %.3g  epi_busy %.3g  tiles %llu  cta_cycles %.3g (sums over CTAs)\n",
              variant, reps + 1, (double)h[0], (double)h[1], (double)h[2], (double)h[3], (double)h[4], h[5], (double)h[6]);
    cudaFree(dstats);
  }
  if (e != cudaSuccess) return fail(nullptr, PROBE_ECUDA, "probe_test_gemm: %s", cudaGetErrorString(e));
  return PROBE_OK;
}

probe_status probe_check(probe_ctx ctx) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  CK(cudaStreamSynchronize(ctx->aux));
  CK(cudaStreamSynchronize(ctx->pf));
  CK(cudaDeviceSynchronize());
  int32_t flags[4];
  CK(cudaMemcpy(flags, ctx->scratch + ctx->sl.flags, sizeof(flags), cudaMemcpyDeviceToHost));
  if (flags[0] & ERR_RECV_OVERFLOW)
    return fail(ctx, PROBE_ECAPACITY, "receive capacity overflow (ranks [%d,%d), recv_capacity=%d)", ctx->cfg.rank_begin,
                ctx->cfg.rank_begin + ctx->cfg.local_ranks, ctx->cfg.recv_capacity);
  if (flags[0] & ERR_Y_RANGE)
    return fail(ctx, PROBE_ESHAPE, "expert output |y| > 65504 does not fit the fp16 Y buffer (D2)");
  if (flags[0]) return fail(ctx, PROBE_ECUDA, "device error word 0x%x", flags[0]);
  return PROBE_OK;
}

const char* probe_last_error(probe_ctx ctx) {
  if (ctx) return ctx->err.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_last_error.c_str();
}

probe_status probe_finalize(probe_ctx ctx) {
  if (!ctx) return PROBE_OK;
  cudaDeviceSynchronize();
  for (int p = 0; p < 2; ++p) {
    cudaEventDestroy(ctx->ev_gate[p]); cudaEventDestroy(ctx->ev_gemm[p]); cudaEventDestroy(ctx->ev_comb[p]);
    cudaEventDestroy(ctx->ev_pred[p]); cudaEventDestroy(ctx->ev_plan[p]); cudaEventDestroy(ctx->ev_slots[p]);
    cudaEventDestroy(ctx->ev_disp[p]);
  }
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->pf) cudaStreamDestroy(ctx->pf);
  if (ctx->pd) cudaStreamDestroy(ctx->pd);
  if (ctx->ev_fwd_start) cudaEventDestroy(ctx->ev_fwd_start);
  if (ctx->ev_pd_done) cudaEventDestroy(ctx->ev_pd_done);
  for (auto e : ctx->prof_ev) cudaEventDestroy(e);
  if (ctx->dbuf) cudaFree(ctx->dbuf);
  delete ctx;
  return PROBE_OK;
}

int64_t probe_launch_count(probe_ctx ctx) { return ctx ? ctx->launches : 0; }

probe_status probe_history_update(probe_ctx ctx, int32_t layer, int32_t reset, int32_t* history, void* stream) {
  if (!ctx || !history) return fail(ctx, PROBE_EINVAL, "probe_history_update: null argument");
  if (ctx->fwd_layer < layer || ((ctx->fwd_layer - layer) > 1))
    return fail(ctx, PROBE_ESTATE, "probe_history_update(%d): counts of that layer are no longer on the board", layer);
  const Dims& d = ctx->d;
  const int32_t* board = reinterpret_cast<const int32_t*>(ctx->local_base[PROBE_BUF_BOARD]) + (((layer & 1) * 2 + 0) * d.G) * d.E;
  k_history<<<(d.G * d.E + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(d.G * d.E, board, history, reset);
  CKL();
  return PROBE_OK;
}

// ---- NEXT-1: online distillation of the predictor residual (R33-R37) ----------
// Workspace for N = local_ranks · max_tokens tokens, Np = N rounded up to 64:
//   z fp32 [N,h] | a bf16 [N,h] | aT [h,Np] | lhat, t fp32 [N,E] | gl bf16 [N,E] | glT [E,Np]
//   | ga fp32 [N,h] | gzT [h,Np] | xT [H,Np] | w2T [h,E] | 6 GEMM schedules
struct DistillLayout {
  size_t z, a, aT, lhat, t, gl, glT, ga, gzT, xT, w2T, part, sched, total;
  uint64_t Np;
};

static DistillLayout distill_layout(const probe_config& c) {
  DistillLayout L{};
  const uint64_t N = static_cast<uint64_t>(c.local_ranks) * c.max_tokens, Np = al(N, 64);
  const uint64_t h = c.res_hidden, E = c.num_experts, H = c.hidden;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += al(bytes, 1024); return r; };
  L.Np = Np;
  L.z = take(N * h * 4);
  L.a = take(N * h * 2);
  L.aT = take(h * Np * 2);
  L.lhat = take(N * E * 4);
  L.t = take(N * E * 4);
  L.gl = take(N * E * 2);
  L.glT = take(E * Np * 2);
  L.ga = take(N * h * 4);
  L.gzT = take(h * Np * 2);
  L.xT = take(H * Np * 2);
  L.w2T = take(h * E * 2);
  L.part = take(static_cast<size_t>(kSplitMax) * std::max(E * h, h * H) * 4);
  L.sched = take(kDistillScheds * sizeof(GemmSched));
  L.total = o;
  return L;
}

probe_status probe_distill_grad(probe_ctx ctx, const void* x, const void* x_next, int32_t T, const void* w_router,
                                const float* b_router, const void* w_res1, const void* w_res2, float* grad_res1,
                                float* grad_res2, double* stats, int32_t fidelity, float* student_logits,
                                float* teacher_logits, void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  if (!x || !x_next || !w_router || !w_res1 || !w_res2 || !grad_res1 || !grad_res2 || !stats)
    return fail(ctx, PROBE_EINVAL, "probe_distill_grad: null pointer");
  if (ctx->cfg.res_hidden <= 0) return fail(ctx, PROBE_ESHAPE, "probe_distill_grad: res_hidden == 0");
  if (ctx->f32()) return fail(ctx, PROBE_ESHAPE, "probe_distill_grad: bf16 only (dtype = PROBE_FP32)");
  if (T < 1 || T > ctx->cfg.max_tokens) return fail(ctx, PROBE_ECAPACITY, "T=%d outside [1, max_tokens]", T);
  cudaStream_t st = static_cast<cudaStream_t>(stream);   // NULL = the legacy default stream
  const DistillLayout DL = distill_layout(ctx->cfg);
  if (!ctx->dbuf) {
    if (capture_id(st) != 0)
      return fail(ctx, PROBE_ESTATE, "probe_distill_grad: first call (workspace allocation) inside stream capture");
    CK(cudaMalloc(&ctx->dbuf, DL.total));
    ctx->dbytes = DL.total;
  }
  const Dims& d = ctx->d;
  const int N = d.GL * T, H = d.H, E = d.E, h = d.h;
  const int Np = static_cast<int>(al(static_cast<uint64_t>(N), 64));
  const int grid = ctx->aux_sms;
  uint8_t* B = ctx->dbuf;
  float* z = reinterpret_cast<float*>(B + DL.z);
  auto* a = reinterpret_cast<__nv_bfloat16*>(B + DL.a);
  auto* aT = reinterpret_cast<__nv_bfloat16*>(B + DL.aT);
  float* lhat = student_logits ? student_logits : reinterpret_cast<float*>(B + DL.lhat);
  float* tl = teacher_logits ? teacher_logits : reinterpret_cast<float*>(B + DL.t);
  auto* gl = reinterpret_cast<__nv_bfloat16*>(B + DL.gl);
  auto* glT = reinterpret_cast<__nv_bfloat16*>(B + DL.glT);
  float* ga = reinterpret_cast<float*>(B + DL.ga);
  auto* gzT = reinterpret_cast<__nv_bfloat16*>(B + DL.gzT);
  auto* xT = reinterpret_cast<__nv_bfloat16*>(B + DL.xT);
  auto* w2T = reinterpret_cast<__nv_bfloat16*>(B + DL.w2T);
  float* part = reinterpret_cast<float*>(B + DL.part);
  GemmSched* sch = reinterpret_cast<GemmSched*>(B + DL.sched);
  const CUtensorMap* mx = ctx->maps.get(x, N, H, 128);
  const CUtensorMap* mxn = ctx->maps.get(x_next, N, H, 128);
  const CUtensorMap* mw = ctx->maps.get(w_router, E, H, 64);
  const CUtensorMap* m1 = ctx->maps.get(w_res1, h, H, 64);
  const CUtensorMap* m2 = ctx->maps.get(w_res2, E, h, 64);
  const CUtensorMap* ma = ctx->maps.get(a, N, h, 128);
  const CUtensorMap* mglT = ctx->maps.get(glT, E, Np, 128);
  const CUtensorMap* maT = ctx->maps.get(aT, h, Np, 64);
  const CUtensorMap* mgl = ctx->maps.get(gl, N, E, 128);
  const CUtensorMap* mw2T = ctx->maps.get(w2T, h, E, 64);
  const CUtensorMap* mgzT = ctx->maps.get(gzT, h, Np, 128);
  const CUtensorMap* mxT = ctx->maps.get(xT, H, Np, 64);
  if (!mx || !mxn || !mw || !m1 || !m2 || !ma || !mglT || !maT || !mgl || !mw2T || !mgzT || !mxT)
    return fail(ctx, PROBE_ECUDA, "tensor map encode failed");
  // Schedules (one launch writes all six).  The two token contractions (K = Np) are split
  // along K when their output has fewer tiles than the grid: split s covers K elements
  // [s·Ks, (s+1)·Ks) into part[s], summed in order by k_sum_partials (deterministic).
  DistillSpecs sp{};
  int ksplit[kDistillScheds], nsplit[kDistillScheds];
  auto spec = [&](int si, int m, int n, int K, float* out, bool allow_split) {
    int S = 1;
    if (allow_split) {
      const int tiles = ((m + 127) / 128) * ((n + 127) / 128);
      S = std::max(1, std::min({kSplitMax, grid / std::max(tiles, 1), K / 512}));
    }
    const int Ks = ((K + S - 1) / S + 63) / 64 * 64;
    S = (K + Ks - 1) / Ks;
    sp.s[si].n = S;
    for (int j = 0; j < S; ++j) {
      sp.s[si].g[j] = mk_group(0, m, 0, 0, EPI_F32, n, n, S > 1 ? part + static_cast<size_t>(j) * m * n : out);
      sp.s[si].g[j].k_off = j * Ks;
    }
    ksplit[si] = S > 1 ? Ks : K;
    nsplit[si] = S;
  };
  spec(0, N, h, H, z, false);            // z = x Ŵ¹ᵀ
  spec(1, N, E, H, lhat, false);         // l̂ = [x | a]·[W | Ŵ²]ᵀ  (K2 = h)
  spec(2, N, E, H, tl, false);           // t = x' Wᵀ
  spec(3, E, h, Np, grad_res2, true);    // ∇Ŵ² = g_lᵀ a
  spec(4, N, h, E, ga, false);           // g_a = g_l Ŵ²
  spec(5, h, H, Np, grad_res1, true);    // ∇Ŵ¹ = g_zᵀ x
  auto gemm = [&](int si, const CUtensorMap& A, const CUtensorMap& B0, const CUtensorMap& B1,
                  const CUtensorMap* A2, int K2) -> probe_status {
    CK(launch_gemm_v(V_128_6_4, A, B0, B1, A, sch + si, ksplit[si], grid, st, A2, K2));
    ++ctx->launches;
    return PROBE_OK;
  };
  auto reduce = [&](int si, float* out, int64_t n) -> probe_status {
    if (nsplit[si] <= 1) return PROBE_OK;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(ctx->num_sms) * 8);
    k_sum_partials<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part, out, n, nsplit[si]);
    CKL();
    return PROBE_OK;
  };
  const dim3 tb(32, 8);
  probe_status r;
  CK(cudaMemsetAsync(stats, 0, 4 * sizeof(double), st));
  k_write_scheds<<<1, 32, 0, st>>>(sch, sp);
  CKL();
  // operands that the backward contracts over tokens: xᵀ [H, Np], Ŵ²ᵀ [h, E]
  k_transpose_bf16<<<dim3((H + 63) / 64, (Np + 63) / 64), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), xT,
                                                                         N, H, Np);
  CKL();
  k_transpose_bf16<<<dim3((h + 63) / 64, (E + 63) / 64), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w_res2),
                                                                        w2T, E, h, E);
  CKL();
  // forward: z = x Ŵ¹ᵀ;  a = bf16(σ(z));  l̂ = [x | a]·[W | Ŵ²]ᵀ (Eq. (P));  t = x' Wᵀ (R33)
  if ((r = gemm(0, *mx, *m1, *m1, nullptr, 0)) != PROBE_OK) return r;
  k_act_fwd<<<dim3((h + 31) / 32, (Np + 31) / 32), tb, 0, st>>>(z, a, aT, N, h, Np);
  CKL();
  if ((r = gemm(1, *mx, *mw, *m2, ma, h)) != PROBE_OK) return r;
  if ((r = gemm(2, *mxn, *mw, *mw, nullptr, 0)) != PROBE_OK) return r;
  // softmax / CE / g_l = q − p / fidelity (R34, R37)
  k_distill_ce<<<(N + 31) / 32, 1024, 0, st>>>(lhat, tl, b_router, N, E, fidelity ? d.k : 0, Np, gl, glT, stats);
  CKL();
  // backward (R34, R35): ∇Ŵ² = g_lᵀ a;  g_a = g_l Ŵ²;  g_z = g_a ⊙ σ'(z);  ∇Ŵ¹ = g_zᵀ x
  if ((r = gemm(3, *mglT, *maT, *maT, nullptr, 0)) != PROBE_OK) return r;
  if ((r = reduce(3, grad_res2, static_cast<int64_t>(E) * h)) != PROBE_OK) return r;
  if ((r = gemm(4, *mgl, *mw2T, *mw2T, nullptr, 0)) != PROBE_OK) return r;
  k_silu_bwd<<<dim3((h + 31) / 32, (Np + 31) / 32), tb, 0, st>>>(ga, z, gzT, N, h, Np);
  CKL();
  if ((r = gemm(5, *mgzT, *mxT, *mxT, nullptr, 0)) != PROBE_OK) return r;
  if ((r = reduce(5, grad_res1, static_cast<int64_t>(h) * H)) != PROBE_OK) return r;
  return PROBE_OK;
}

probe_status probe_distill_apply(probe_ctx ctx, float* master, const float* grad, void* w, int64_t n, float scale,
                                 void* stream) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  if (!master || !grad || !w || n < 0) return fail(ctx, PROBE_EINVAL, "probe_distill_apply: bad arguments");
  if (n == 0) return PROBE_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(ctx->num_sms) * 8);
  k_sgd<<<static_cast<unsigned>(blocks), 256, 0, st>>>(master, grad, static_cast<__nv_bfloat16*>(w), n, scale);
  CKL();
  return PROBE_OK;
}

probe_status probe_set_option(probe_ctx ctx, int32_t option, int64_t value) {
  if (!ctx) return fail(nullptr, PROBE_EINVAL, "null ctx");
  switch (option) {
    case PROBE_OPT_EP_EMULATION: ctx->ep_emulation = value != 0; return PROBE_OK;
    case PROBE_OPT_UNFUSED_TOPK: ctx->unfused = value != 0; return PROBE_OK;
    case PROBE_OPT_FUSED_EPILOGUE_TOPK: ctx->fused_epi_topk = value != 0; return PROBE_OK;
    case PROBE_OPT_PAIR_GEMM: ctx->pair_gemm = value != 0; return PROBE_OK;
    case PROBE_OPT_AUX_START:
      if (value < 0 || value > 1) return fail(ctx, PROBE_EINVAL, "aux start %lld not in {0, 1}", (long long)value);
      ctx->aux_start = static_cast<int>(value);
      return PROBE_OK;
    case PROBE_OPT_PRED_PAIR: ctx->pred_pair = value != 0; return PROBE_OK;
    case PROBE_OPT_L2_HINTS:
      if (value < 0 || value > 0x77) return fail(ctx, PROBE_EINVAL, "L2 hint mask 0x%llx", (long long)value);
      ctx->l2hint = static_cast<int>(value);
      return PROBE_OK;
    case PROBE_OPT_PRED_MAXREG:
      if (value != 0 && value != 192) return fail(ctx, PROBE_EINVAL, "predictor register cap %lld not in {0, 192}", (long long)value);
      ctx->pred_maxreg = static_cast<int>(value);
      return PROBE_OK;
    case PROBE_OPT_AUX_SMS:
      if (value < 1 || value > ctx->num_sms) return fail(ctx, PROBE_EINVAL, "aux SM cap %lld out of range", (long long)value);
      ctx->aux_sms = static_cast<int>(value);
      return PROBE_OK;
  }
  return fail(ctx, PROBE_EINVAL, "unknown option %d", option);
}

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

probe_status probe_ipc_export(const void* dev_ptr, uint8_t handle[64], uint64_t* offset) {
  probe_ctx ctx = nullptr;
  if (!dev_ptr || !handle || !offset) return fail(nullptr, PROBE_EINVAL, "probe_ipc_export: null argument");
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) return fail(nullptr, PROBE_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (reinterpret_cast<PFN_getAddressRange>(fn)(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(nullptr, PROBE_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &h, 64);
  *offset = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
  return PROBE_OK;
}

probe_status probe_ipc_import(const uint8_t handle[64], uint64_t offset, uint64_t* dev_ptr) {
  probe_ctx ctx = nullptr;
  if (!handle || !dev_ptr) return fail(nullptr, PROBE_EINVAL, "probe_ipc_import: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = reinterpret_cast<uint64_t>(p) + offset;
  return PROBE_OK;
}

probe_status probe_ipc_close(uint64_t dev_ptr_base) {
  probe_ctx ctx = nullptr;
  CK(cudaIpcCloseMemHandle(reinterpret_cast<void*>(dev_ptr_base)));
  return PROBE_OK;
}

probe_status probe_profile(probe_ctx ctx, int32_t n) {
  if (!ctx || n < 0) return fail(ctx, PROBE_EINVAL, "probe_profile: bad arguments");
  CK(cudaDeviceSynchronize());
  for (auto e : ctx->prof_ev) cudaEventDestroy(e);
  ctx->prof_ev.assign(static_cast<size_t>(n) * (PROBE_NPHASE + 1), nullptr);
  for (auto& e : ctx->prof_ev) CK(cudaEventCreate(&e));
  ctx->prof_max = n;
  ctx->prof_n = 0;
  return PROBE_OK;
}

probe_status probe_profile_read(probe_ctx ctx, float* ms, int32_t* n_out) {
  if (!ctx || !n_out) return fail(ctx, PROBE_EINVAL, "probe_profile_read: bad arguments");
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < ctx->prof_n; ++i) {
    cudaEvent_t* ev = &ctx->prof_ev[static_cast<size_t>(i) * (PROBE_NPHASE + 1)];
    // phase j spans marks j..j+1; TOTAL spans the first to the last mark
    // marks 0..PROBE_PH_TOTAL on the main stream; the last event = pre-dispatch done (side stream)
    int order[PROBE_NPHASE][2];
    for (int j = 0; j < PROBE_PH_TOTAL; ++j) { order[j][0] = j; order[j][1] = j + 1; }
    order[PROBE_PH_TOTAL][0] = 0;
    order[PROBE_PH_TOTAL][1] = PROBE_PH_TOTAL;
    order[PROBE_PH_PREDISPATCH][0] = 0;
    order[PROBE_PH_PREDISPATCH][1] = PROBE_PH_PREDISPATCH;
    for (int j = 0; j < PROBE_NPHASE; ++j) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[order[j][0]], ev[order[j][1]]));
      if (ms) ms[i * PROBE_NPHASE + j] = t;
    }
  }
  *n_out = ctx->prof_n;
  return PROBE_OK;
}

}  // extern "C"
