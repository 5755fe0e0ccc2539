"""Online distillation driver for the lookahead predictor's residual.

P:387-390: the residual MLP (Ŵ¹, Ŵ²) of Eq. (P) is trained on the live request stream by
minimising the cross-entropy to the ground-truth router's probabilities; the frozen prior
stays untouched.  Every arithmetic step runs in libprobe.so (probe_distill_grad /
probe_distill_apply); this class only owns the buffers, and — when the predictor is
replicated over several processes — sums the gradients and statistics with one
all-reduce (the one real exchange of data-parallel training), then applies the step with
the GLOBAL token count (R34, R36).
"""
from __future__ import annotations

from typing import Optional

import torch

from .runtime import ProbeRuntime


class PredictorDistiller:
    """fp32 master copies of Ŵ¹ [h,H], Ŵ² [E,h] plus the bf16 weights the product path reads.

    `w_res1` / `w_res2` (bf16, device) are updated in place after each step, so a runtime
    that predicts with them sees the distilled residual immediately.
    """

    def __init__(self, rt: ProbeRuntime, w_res1: torch.Tensor, w_res2: torch.Tensor,
                 master1: Optional[torch.Tensor] = None, master2: Optional[torch.Tensor] = None):
        self.rt = rt
        self.w1, self.w2 = w_res1, w_res2
        self.m1 = (w_res1.float() if master1 is None else master1).contiguous().clone()
        self.m2 = (w_res2.float() if master2 is None else master2).contiguous().clone()
        self.g1 = torch.empty_like(self.m1)
        self.g2 = torch.empty_like(self.m2)
        self.stats = torch.empty(4, dtype=torch.float64, device=w_res1.device)

    def grad(self, x, x_next, w_router, b_router=None, student_logits=None, teacher_logits=None,
             fidelity: bool = True, stream=None):
        self.rt.distill_grad(x, x_next, w_router, b_router, self.w1, self.w2, self.g1, self.g2, self.stats,
                             student_logits, teacher_logits, fidelity, stream)

    def step(self, x, x_next, w_router, b_router=None, lr: float = 1e-2, group=None, stream=None,
             want_metrics: bool = True) -> Optional[dict]:
        """One distillation step on this process's GL·T tokens.  Returns the batch metrics
        (a device→host read of four numbers) unless want_metrics=False."""
        self.grad(x, x_next, w_router, b_router, fidelity=want_metrics, stream=stream)
        n_total = float(x.numel() // x.shape[-1])
        if group is not None:
            import torch.distributed as dist
            n = torch.tensor([n_total], dtype=torch.float64, device=self.stats.device)
            for t in (self.g1, self.g2, self.stats, n):
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            n_total = float(n.item())
        scale = -lr / n_total
        self.rt.distill_apply(self.m1, self.g1, self.w1, scale, stream)
        self.rt.distill_apply(self.m2, self.g2, self.w2, scale, stream)
        return metrics(self.stats, n_total, self.rt.cfg.k) if want_metrics else None


def metrics(stats: torch.Tensor, n_tokens: float, k: int) -> dict:
    """R37: mean CE, top-K accuracy, top-half-K hit rate, 2×top-K recall from the sums."""
    s = stats.double().cpu().tolist()
    return {"loss": s[0] / n_tokens, "topk_acc": s[1] / (n_tokens * k),
            "top_half_k_hit": s[2] / (n_tokens * ((k + 1) // 2)), "twice_topk_recall": s[3] / (n_tokens * k)}
