"""GPU: the multi-process EP path for real — two processes on ONE B200, each hosting one
logical rank (G=2), symmetric buffers shared through CUDA IPC handles exchanged over
torch.distributed (gloo), cross-process device barriers on the signal pads.  Results are
compared with the fp64 oracle exactly as in the single-process tests."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, zipf):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch.distributed as dist
    import probe_inputs as pi
    from paper_2602_00509_b200 import ProbeConfig
    from paper_2602_00509_b200.dist import make_runtime_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    sh = pi.C0
    G, E, k, H, F, T = sh.G, sh.E, sh.k, sh.H, sh.F, sh.T
    EL = E // G
    cfg = ProbeConfig(G=G, E=E, k=k, H=H, F=F, T=T, h=sh.h, rank_begin=rank, local_ranks=1,
                      replica_budget=3, alpha_ps=1, beta_ps=0, n_sat=0)
    rt = make_runtime_distributed(cfg, dev)
    L0 = pi.layer_inputs(sh, 0, 0, zipf, ranks=[rank], device=dev)
    L1 = pi.layer_inputs(sh, 0, 1, zipf, ranks=[rank], device=dev)
    W = [pi.router_weight(sh, p, device=dev) for p in (0, 1)]
    w13, w2 = [], []
    for p in (0, 1):
        a, b = pi.expert_weights(sh, p, experts=range(rank * EL, (rank + 1) * EL), device=dev)
        w13.append(a)
        w2.append(b)
    r1, r2 = pi.predictor_residual(sh, 1, device=dev)
    out = [torch.empty(1, T, H, device=dev) for _ in (0, 1)]
    ids = [torch.empty(1, T, k, dtype=torch.int32, device=dev) for _ in (0, 1)]
    reps = torch.empty(G, 3, dtype=torch.int32, device=dev)
    quota = torch.empty(G, E, G, dtype=torch.int32, device=dev)
    pc = torch.empty(G, E, dtype=torch.int32, device=dev)
    win = torch.full((G,), 10 ** 9, dtype=torch.int64, device=dev)
    rt.forward(0, L0.x, W[0], None, w13[0], w2[0], out[0], topk_ids=ids[0])
    rt.predict(1, L0.x, W[1], None, r1, r2, pred_counts=pc)
    rt.plan(1, win, replicas=reps, quota=quota)
    rt.prefetch(1, w13[1], w2[1], phase=0)
    rt.forward(1, L1.x, W[1], None, w13[1], w2[1], out[1], use_plan=True, topk_ids=ids[1])
    rt.check()
    torch.cuda.synchronize()
    q.put((rank, [o.cpu().numpy() for o in out], [i.cpu().numpy() for i in ids], pc.cpu().numpy(),
           reps.cpu().numpy(), quota.cpu().numpy()))
    dist.barrier()
    rt.close()
    dist.destroy_process_group()


def test_two_processes_one_gpu_ipc():
    sys.path.insert(0, HERE)
    import oracle as O
    import probe_inputs as pi
    from layer_harness import CaseCfg, run_oracle
    zipf = 1.5
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, zipf)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in ps)
    sh = pi.C0
    case = CaseCfg(sh, zipf_s=zipf)
    inputs = dict(L0=pi.layer_inputs(sh, 0, 0, zipf), L1=pi.layer_inputs(sh, 0, 1, zipf),
                  W=[pi.router_weight(sh, p) for p in (0, 1)], b=[None, None],
                  w13=[pi.expert_weights(sh, p)[0] for p in (0, 1)], w2=[pi.expert_weights(sh, p)[1] for p in (0, 1)])
    inputs["r1"], inputs["r2"] = pi.predictor_residual(sh, 1)
    orc = run_oracle(case, inputs)
    plan = orc["plan"]
    assert any(plan.replicas)
    for rank, outs, ids, pc, reps, quota in res:
        assert np.array_equal(pc, orc["nhat"])
        assert np.array_equal(quota, plan.quota)
        for L in (0, 1):
            ref = orc["ref"][L]
            assert np.array_equal(ids[L][0], ref["ids"][rank])
            rms = np.sqrt(np.mean(np.concatenate([o.reshape(-1) for o in ref["out"]]) ** 2))
            assert np.abs(outs[L][0] - ref["out"][rank]).max() <= 2e-2 * rms
