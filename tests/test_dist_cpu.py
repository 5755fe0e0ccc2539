"""Multi-process host logic on CPU (gloo, world_size 2): rank partition, handle exchange
through torch.distributed, and the [NSYM][G] peer-table construction probe_init expects."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2602_00509_b200 import _lib
from paper_2602_00509_b200.dist import build_peer_table, rank_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2602_00509_b200.dist import exchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = 8
    r0, gl = rank_range(G, world, rank)
    # fake "exported handles": (bytes, offset) per buffer kind, tagged by process
    mine = [(bytes([rank]) * 64, 1024 * b) for b in range(_lib.PROBE_NSYM)]
    allh = exchange(mine)
    bases = [[0x10000000 * (p + 1) + 0x100000 * b for b in range(_lib.PROBE_NSYM)] for p in range(world)]
    sizes = [4096 * (b + 1) for b in range(_lib.PROBE_NSYM)]
    table = build_peer_table(bases, sizes, G)
    q.put((rank, r0, gl, [h[0][0][0] for h in allh], table))
    dist.destroy_process_group()


def test_gloo_exchange_and_peer_table():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, r0, gl, tags, table in res:
        assert (r0, gl) == (rank * 4, 4)
        assert tags == [0, 1]                       # every process saw every process's handles in order
        for b in range(_lib.PROBE_NSYM):
            for r in range(8):
                p = r // 4
                assert table[b][r] == 0x10000000 * (p + 1) + 0x100000 * b + (r % 4) * 4096 * (b + 1)
    assert res[0][4] == res[1][4]                   # identical tables on every process


def test_rank_range_rejects_uneven():
    with pytest.raises(ValueError):
        rank_range(8, 3, 0)


class _FakeRuntime:
    """CPU test double for the two distillation calls (the gradient is a rank-tagged
    constant, the update the R36 formula), so only PredictorDistiller's host logic —
    the SUM all-reduce of gradients / statistics / token counts and the global lr/N
    scale — is under test."""

    class cfg:
        k = 2

    def __init__(self, rank):
        self.rank = rank

    def distill_grad(self, x, x_next, w_router, b_router, w1, w2, g1, g2, stats, sl, tl, fidelity, stream):
        g1.fill_(float(self.rank + 1))
        g2.fill_(float(10 * (self.rank + 1)))
        stats.copy_(torch.tensor([1.5 * (self.rank + 1), 3.0, 2.0, 4.0], dtype=torch.float64))

    def distill_apply(self, master, grad, w, scale, stream):
        master.add_(grad, alpha=scale)
        w.copy_(master.to(w.dtype))


def _distill_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2602_00509_b200.distill import PredictorDistiller
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w1 = torch.zeros(4, 8, dtype=torch.bfloat16)
    w2 = torch.zeros(6, 4, dtype=torch.bfloat16)
    d = PredictorDistiller(_FakeRuntime(rank), w1, w2)
    x = torch.zeros(3 + rank, 8)                   # 3 and 4 tokens: global N = 7
    met = d.step(x, x, None, lr=0.7, group=dist.group.WORLD)
    q.put((rank, d.m1.clone(), d.m2.clone(), w1.clone(), met))
    dist.destroy_process_group()


def test_gloo_distiller_allreduce():
    import torch
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_distill_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m1, m2, w1, met in res:
        assert torch.allclose(m1, torch.full_like(m1, -0.7 / 7 * 3))      # Σ_ranks ∇Ŵ¹ = 1 + 2
        assert torch.allclose(m2, torch.full_like(m2, -0.7 / 7 * 30))     # Σ_ranks ∇Ŵ² = 10 + 20
        assert torch.equal(w1, m1.to(torch.bfloat16))
        assert abs(met["loss"] - (1.5 + 3.0) / 7) < 1e-12
        assert abs(met["topk_acc"] - 6.0 / (7 * 2)) < 1e-12
    assert torch.equal(res[0][1], res[1][1])                               # replicas stay identical
