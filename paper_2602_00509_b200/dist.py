"""One process per GPU: symmetric buffers shared through CUDA IPC handles exchanged over
torch.distributed (NCCL on GPUs, gloo in CPU tests).  Host-side plumbing only.

Process p (of N) hosts logical ranks [p·G/N, (p+1)·G/N).  Each process allocates one
tensor per symmetric buffer kind (its G/N ranks contiguous, stride = per-rank bytes),
exports (IPC handle, offset) per kind, all-gathers them, maps the peers' allocations,
and builds the [NSYM][G] peer table probe_init expects.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import torch

from . import _lib
from ._lib import check
from .runtime import ProbeConfig, ProbeRuntime, _aligned, workspace_sizes


def rank_range(G: int, world: int, proc: int):
    if G % world:
        raise ValueError(f"EP size {G} not divisible by {world} processes")
    gl = G // world
    return proc * gl, gl


def build_peer_table(bases: Sequence[Sequence[int]], sizes: Sequence[int], G: int) -> List[List[int]]:
    """bases[p][b] = address (as mapped here) of process p's buffer b; returns table[b][r]."""
    world = len(bases)
    gl = G // world
    return [[int(bases[r // gl][b]) + (r % gl) * int(sizes[b]) for r in range(G)] for b in range(_lib.PROBE_NSYM)]


def export_handles(tensors: Sequence[torch.Tensor]):
    lib = _lib.load()
    out = []
    for t in tensors:
        h = (C.c_uint8 * 64)()
        off = C.c_uint64(0)
        check("probe_ipc_export", lib.probe_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
        out.append((bytes(h), int(off.value)))
    return out


def import_handles(handles, opened: List[int] = None):
    """Map peer allocations; the mapped bases (address − offset) are appended to `opened` so
    the caller can unmap them (close_handles) when the runtime is closed."""
    lib = _lib.load()
    ptrs = []
    for (h, off) in handles:
        arr = (C.c_uint8 * 64).from_buffer_copy(h)
        p = C.c_uint64(0)
        check("probe_ipc_import", lib.probe_ipc_import(arr, off, C.byref(p)))
        ptrs.append(int(p.value))
        if opened is not None:
            opened.append(int(p.value) - int(off))
    return ptrs


def close_handles(bases: Sequence[int]):
    lib = _lib.load()
    for b in bases:
        check("probe_ipc_close", lib.probe_ipc_close(C.c_uint64(b)))


def exchange(obj, group=None):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def make_runtime_distributed(cfg: ProbeConfig, device, group=None) -> ProbeRuntime:
    import torch.distributed as dist
    world = dist.get_world_size(group)
    proc = dist.get_rank(group)
    r0, gl = rank_range(cfg.G, world, proc)
    if cfg.rank_begin != r0 or cfg.local_ranks != gl:
        raise ValueError("cfg.rank_begin/local_ranks do not match this process")
    sizes = workspace_sizes(cfg)
    sym = [_aligned(sizes[b] * gl, device) for b in range(_lib.PROBE_NSYM)]
    for b in (_lib.BUF_BOARD, _lib.BUF_SIGNAL):
        sym[b].zero_()
    torch.cuda.synchronize(device)
    mine = export_handles(sym)
    allh = exchange(mine, group)
    bases, opened = [], []
    for p in range(world):
        if p == proc:
            bases.append([t.data_ptr() for t in sym])
        else:
            bases.append(import_handles(allh[p], opened))
    table = build_peer_table(bases, sizes, cfg.G)
    dist.barrier(group)
    rt = ProbeRuntime(cfg, device, peer_tables=table, sym_buffers=sym)
    rt.on_close(lambda: close_handles(opened))   # unmap the peers' allocations with the context
    return rt
