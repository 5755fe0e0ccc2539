"""Multi-process host logic on CPU (gloo, world_size 2): rank partition, handle exchange
through torch.distributed, and the [NSYM][G] peer-table construction probe_init expects."""
import os
import socket

import pytest
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
