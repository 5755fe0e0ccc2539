"""Python binding of the PROBE C-ABI: device memory from PyTorch, calls into libprobe.so.

PyTorch supplies device memory (symmetric buffers, scratch), streams and — for
multi-process runs — the process group used to exchange peer handles.  No
arithmetic of the method happens here.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional

import torch

from . import _lib
from ._lib import check, probe_config


@dataclasses.dataclass
class ProbeConfig:
    G: int
    E: int
    k: int
    H: int
    F: int
    T: int                     # max tokens per rank
    h: int = 0                 # predictor residual width (0 = prior only)
    rank_begin: int = 0
    local_ranks: int = 0       # 0 ⇒ all G ranks in this process (single-GPU emulation)
    recv_capacity: int = 0     # 0 ⇒ worst case T·G·min(k, E/G + 3)
    replica_budget: int = 3
    kmax: int = 16
    n_sat: int = 0
    alpha_ps: int = 1
    beta_ps: int = 0
    bw_bytes_per_us: int = 770_000
    capacity_factor: float = 0.0   # >0 ⇒ recv_capacity = factor · T·k (rounded up to 128)
    dtype: str = "bf16"            # "bf16" (product path, tcgen05) or "fp32" (parity path, SIMT fp32 GEMMs)
    dedup_wire: bool = False       # one wire row per unique (token, dest) + R25 partial-sum combine
    predispatch: bool = False      # NEXT-4: pre-dispatch to predicted experts' home ranks during the gate
    fuse_gate_predictor: bool = False  # gate GEMM also computes the next layer's prior and Ŵ1 activation

    def __post_init__(self):
        if self.local_ranks == 0:
            self.local_ranks = self.G - self.rank_begin
        if self.recv_capacity == 0:
            if self.capacity_factor > 0:
                cap = int(self.capacity_factor * self.T * self.k)
            else:
                cap = self.T * self.G * min(self.k, self.E // self.G + 3)
            self.recv_capacity = (cap + 127) // 128 * 128

    def to_c(self) -> probe_config:
        return probe_config(self.G, self.rank_begin, self.local_ranks, self.E, self.k, self.H, self.F, self.h,
                            self.T, self.recv_capacity, self.replica_budget, self.kmax, self.n_sat,
                            _lib.DTYPES[self.dtype], int(self.dedup_wire), int(self.predispatch),
                            int(self.fuse_gate_predictor), self.alpha_ps, self.beta_ps,
                            self.bw_bytes_per_us, self.expert_bytes)

    @property
    def torch_dtype(self):
        return torch.float32 if self.dtype == "fp32" else torch.bfloat16

    @property
    def expert_bytes(self) -> int:
        """𝒲 = 3·H·F·sizeof(dtype): W13 [2F,H] + W2 [H,F]."""
        return 3 * self.H * self.F * (4 if self.dtype == "fp32" else 2)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(s=None):
    s = torch.cuda.current_stream() if s is None else s
    return C.c_void_p(s.cuda_stream)


def _aligned(nbytes: int, device) -> torch.Tensor:
    """uint8 device tensor whose data_ptr is 1024-byte aligned (view into a slightly larger block)."""
    raw = torch.empty(nbytes + 1024, dtype=torch.uint8, device=device)
    off = (-raw.data_ptr()) % 1024
    return raw[off:off + nbytes]


def workspace_sizes(cfg: ProbeConfig) -> List[int]:
    lib = _lib.load()
    arr = (C.c_uint64 * _lib.PROBE_NBUF)()
    c = cfg.to_c()
    check("probe_workspace", lib.probe_workspace(C.byref(c), arr))
    return list(arr)


class ProbeRuntime:
    """One probe_ctx: the logical ranks [rank_begin, rank_begin + local_ranks) of this process.

    peer_tables: optional [NSYM][G] list of device addresses (multi-process: exchanged via
    torch.distributed); by default all G ranks are local (single-GPU emulation).
    """

    def __init__(self, cfg: ProbeConfig, device="cuda", peer_tables: Optional[List[List[int]]] = None,
                 sym_buffers: Optional[List[torch.Tensor]] = None):
        self.cfg = cfg
        self.device = torch.device(device)
        self.lib = _lib.load()
        self.sizes = workspace_sizes(cfg)
        G, GL, R0 = cfg.G, cfg.local_ranks, cfg.rank_begin
        if sym_buffers is None:
            sym_buffers = [_aligned(self.sizes[b] * GL, self.device) for b in range(_lib.PROBE_NSYM)]
            for b in (_lib.BUF_BOARD, _lib.BUF_SIGNAL):
                sym_buffers[b].zero_()
        self.sym = sym_buffers
        self.scratch = _aligned(self.sizes[_lib.BUF_SCRATCH], self.device)
        if peer_tables is None:
            if GL != G:
                raise ValueError("peer_tables required when this process does not host all ranks")
            peer_tables = [[self.sym[b].data_ptr() + (r - R0) * self.sizes[b] for r in range(G)]
                           for b in range(_lib.PROBE_NSYM)]
        flat = (C.c_uint64 * (_lib.PROBE_NSYM * G))(*[int(v) for row in peer_tables for v in row])
        self.ctx = C.c_void_p()
        c = cfg.to_c()
        check("probe_init", self.lib.probe_init(C.byref(c), flat, _ptr(self.scratch), C.byref(self.ctx)))

    # ------------------------------------------------------------------ views of symmetric buffers
    def sym_view(self, buf: int, local_rank: int, dtype, shape):
        n = int(torch.Size(shape).numel()) * torch.empty(0, dtype=dtype).element_size()
        base = self.sym[buf][local_rank * self.sizes[buf]: local_rank * self.sizes[buf] + n]
        return base.view(dtype).view(shape)

    def replica_slots(self, local_rank: int):
        c = self.cfg
        w13 = self.sym_view(_lib.BUF_REP_W13, local_rank, c.torch_dtype, (6, 2 * c.F, c.H))
        w2 = self.sym_view(_lib.BUF_REP_W2, local_rank, c.torch_dtype, (6, c.H, c.F))
        return w13, w2

    # ------------------------------------------------------------------ API
    def forward(self, layer: int, x, w_router, b_router, w13, w2, out, use_plan: bool = False,
                topk_ids=None, topk_w=None, stream=None):
        T = x.shape[-2]
        st = self.lib.probe_moe_forward(self.ctx, layer, _ptr(x), T, _ptr(w_router), _ptr(b_router), _ptr(w13),
                                        _ptr(w2), int(use_plan), _ptr(out), int(out.dtype == torch.float32),
                                        _ptr(topk_ids), _ptr(topk_w), _stream(stream))
        check("probe_moe_forward", st, self.ctx)

    def predict(self, next_layer: int, x, w_router_next, b_router_next=None, w_res1=None, w_res2=None,
                pred_counts=None, pred_logits=None, stream=None):
        T = x.shape[-2]
        s = None if stream is None else _stream(stream)
        st = self.lib.probe_predict(self.ctx, next_layer, _ptr(x), T, _ptr(w_router_next), _ptr(b_router_next),
                                    _ptr(w_res1), _ptr(w_res2), _ptr(pred_counts), _ptr(pred_logits), s)
        check("probe_predict", st, self.ctx)

    def predict_prepare(self, next_layer: int, w_router_next, w_res1=None):
        st = self.lib.probe_predict_prepare(self.ctx, next_layer, _ptr(w_router_next), _ptr(w_res1))
        check("probe_predict_prepare", st, self.ctx)

    def plan(self, next_layer: int, window_ns, pred_counts=None, replicas=None, quota=None, stats=None,
             stream=None):
        s = None if stream is None else _stream(stream)
        st = self.lib.probe_plan(self.ctx, next_layer, _ptr(pred_counts), _ptr(window_ns), _ptr(replicas),
                                 _ptr(quota), _ptr(stats), s)
        check("probe_plan", st, self.ctx)

    def prefetch(self, next_layer: int, w13_next=None, w2_next=None, phase: int = 0, stream=None):
        st = self.lib.probe_prefetch(self.ctx, next_layer, _ptr(w13_next), _ptr(w2_next), phase,
                                     _stream(stream) if phase == 1 else None)
        check("probe_prefetch", st, self.ctx)

    def debug_layout(self, counts=None, split_cum=None, route=None, group_rows=None, replicas=None,
                     stream=None):
        st = self.lib.probe_debug_layout(self.ctx, _ptr(counts), _ptr(split_cum), _ptr(route), _ptr(group_rows),
                                         _ptr(replicas), _stream(stream))
        check("probe_debug_layout", st, self.ctx)

    def prefetch_kib(self, stream=None):
        """(part 1, part 2) KiB of replica weights pushed so far (split-phase accounting)."""
        out = torch.zeros(2, dtype=torch.int32, device=self.device)
        check("probe_debug_prefetch", self.lib.probe_debug_prefetch(self.ctx, _ptr(out), _stream(stream)), self.ctx)
        v = out.cpu()
        return int(v[0]), int(v[1])

    def window(self, window_ns, attention_ns: int = 0, fallback_ns: int = 0, stream=None):
        """probe_window (R26): window_ns[G] (device int64) ← measured per-rank GEMM window + attention."""
        s = None if stream is None else _stream(stream)
        st = self.lib.probe_window(self.ctx, int(attention_ns), int(fallback_ns), _ptr(window_ns), s)
        check("probe_window", st, self.ctx)

    def flags(self, stream=None):
        """Device status words (probe_debug_flags): error, suspend, part-1 KiB, part-2 KiB,
        static-EP fallbacks, ... (8 int32)."""
        out = torch.zeros(8, dtype=torch.int32, device=self.device)
        check("probe_debug_flags", self.lib.probe_debug_flags(self.ctx, _ptr(out), _stream(stream)), self.ctx)
        return [int(v) for v in out.cpu()]

    def check(self):
        check("probe_check", self.lib.probe_check(self.ctx), self.ctx)

    def profile(self, n: int):
        check("probe_profile", self.lib.probe_profile(self.ctx, n), self.ctx)

    def profile_read(self):
        """→ float32 tensor [n_forwards, PROBE_NPHASE] of milliseconds (synchronises)."""
        n = C.c_int32(0)
        check("probe_profile_read", self.lib.probe_profile_read(self.ctx, None, C.byref(n)), self.ctx)
        out = torch.zeros(max(n.value, 1), _lib.PROBE_NPHASE, dtype=torch.float32)
        check("probe_profile_read", self.lib.probe_profile_read(self.ctx, C.c_void_p(out.data_ptr()), C.byref(n)),
              self.ctx)
        return out[:n.value]

    def history_update(self, layer: int, history, reset: bool = False, stream=None):
        st = self.lib.probe_history_update(self.ctx, layer, int(reset), _ptr(history), _stream(stream))
        check("probe_history_update", st, self.ctx)

    def distill_grad(self, x, x_next, w_router, b_router, w_res1, w_res2, grad_res1, grad_res2, stats,
                     student_logits=None, teacher_logits=None, fidelity: bool = True, stream=None):
        """probe_distill_grad (NEXT-1): loss / fidelity sums → stats, ∂/∂Ŵ¹, ∂/∂Ŵ²."""
        T = x.shape[-2]
        st = self.lib.probe_distill_grad(self.ctx, _ptr(x), _ptr(x_next), T, _ptr(w_router), _ptr(b_router),
                                         _ptr(w_res1), _ptr(w_res2), _ptr(grad_res1), _ptr(grad_res2), _ptr(stats),
                                         int(fidelity), _ptr(student_logits), _ptr(teacher_logits),
                                         _stream(stream))
        check("probe_distill_grad", st, self.ctx)

    def distill_apply(self, master, grad, w, scale: float, stream=None):
        """probe_distill_apply (R36): master += scale·grad, w = bf16(master)."""
        st = self.lib.probe_distill_apply(self.ctx, _ptr(master), _ptr(grad), _ptr(w), master.numel(),
                                          float(scale), _stream(stream))
        check("probe_distill_apply", st, self.ctx)

    def set_option(self, option: int, value: int):
        check("probe_set_option", self.lib.probe_set_option(self.ctx, option, int(value)), self.ctx)

    def launches(self) -> int:
        return int(self.lib.probe_launch_count(self.ctx))

    def on_close(self, fn):
        """Register a callback run once after the context is finalized (e.g. IPC unmapping)."""
        self._closers = getattr(self, "_closers", []) + [fn]

    def close(self):
        if self.ctx:
            self.lib.probe_finalize(self.ctx)
            self.ctx = C.c_void_p()
            for fn in getattr(self, "_closers", []):
                fn()
            self._closers = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def test_gemm(A: torch.Tensor, B: torch.Tensor, groups: List[List[int]], N: int, mode: int,
              C_out: torch.Tensor, stream=None):
    """Grouped GEMM through the tcgen05 kernel (test hook of the C-ABI)."""
    lib = _lib.load()
    flat = (C.c_int32 * (4 * len(groups)))(*[int(v) for g in groups for v in g])
    st = lib.probe_test_gemm(_ptr(A), A.shape[0], _ptr(B), B.shape[0], A.shape[1], N, flat, len(groups), mode,
                             _ptr(C_out), _stream(stream))
    check("probe_test_gemm", st)


def bench_gemm(A: torch.Tensor, B: torch.Tensor, groups: List[List[int]], N: int, mode: int, C_out: torch.Tensor,
               variant: int = -1, reps: int = 10, stream=None) -> float:
    """Mean milliseconds of one grouped-GEMM launch (variant per probe.h), `reps` back-to-back launches."""
    lib = _lib.load()
    flat = (C.c_int32 * (4 * len(groups)))(*[int(v) for g in groups for v in g])
    ms = C.c_float(0.0)
    st = lib.probe_bench_gemm(_ptr(A), A.shape[0], _ptr(B), B.shape[0], A.shape[1], N, flat, len(groups), mode,
                              variant, reps, C.byref(ms), _ptr(C_out), _stream(stream))
    check("probe_bench_gemm", st)
    return float(ms.value)
