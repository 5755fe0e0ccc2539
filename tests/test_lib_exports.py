"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/probe.h declares, validates configs, and contains tcgen05/TMA SASS."""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

from paper_2602_00509_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "probe.h")).read()
    declared = set(re.findall(r"\b(probe_[a-z_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for s in declared:
        assert re.search(rf"\bT {s}$", nm, re.M), s
        assert hasattr(lib, s)


def test_workspace_and_validation(lib):
    from paper_2602_00509_b200 import ProbeConfig, workspace_sizes
    cfg = ProbeConfig(G=8, E=128, k=8, H=2048, F=768, T=8192, h=512, capacity_factor=4.0)
    sz = workspace_sizes(cfg)
    assert sz[_lib.BUF_RECV] == cfg.recv_capacity * 2048 * 2
    assert sz[_lib.BUF_Y] == cfg.recv_capacity * 2048 * 2          # fp16 Y (D2)
    assert sz[_lib.BUF_REP_W13] == 6 * 2 * 768 * 2048 * 2
    assert all(s % 1024 == 0 for s in sz)
    # invalid configs are rejected synchronously with a message (no GPU needed)
    bad = cfg.to_c()
    bad.num_experts = 100      # not divisible by G
    arr = (C.c_uint64 * 7)()
    st = lib.probe_init(C.byref(bad), arr, C.c_void_p(1024), C.byref(C.c_void_p()))
    assert st == 2 and b"divisible" in lib.probe_last_error(None)
    bad = cfg.to_c()
    bad.replica_budget = 4     # at most three redundant experts per rank
    st = lib.probe_init(C.byref(bad), arr, C.c_void_p(1024), C.byref(C.c_void_p()))
    assert st == 3
    bad = cfg.to_c()
    bad.expert_bytes = 1
    assert lib.probe_init(C.byref(bad), arr, C.c_void_p(1024), C.byref(C.c_void_p())) == 1
    bad = cfg.to_c()
    bad.dtype = 2              # only PROBE_BF16 / PROBE_FP32
    assert lib.probe_init(C.byref(bad), arr, C.c_void_p(1024), C.byref(C.c_void_p())) == 1


def test_fuse_gate_predictor_config(lib):
    """probe_config.fuse_gate_predictor: its double-buffered prior / activation and the
    concatenated [W_L ; W_{L+1} ; Ŵ1] operand enlarge the scratch; unsupported shapes and
    dtypes are rejected at init; probe_predict_prepare checks its arguments on the host."""
    from paper_2602_00509_b200 import ProbeConfig, workspace_sizes
    base = ProbeConfig(G=8, E=128, k=8, H=2048, F=768, T=8192, h=512, capacity_factor=4.0)
    fused = ProbeConfig(G=8, E=128, k=8, H=2048, F=768, T=8192, h=512, capacity_factor=4.0,
                        fuse_gate_predictor=True)
    extra = workspace_sizes(fused)[_lib.BUF_SCRATCH] - workspace_sizes(base)[_lib.BUF_SCRATCH]
    M = 8 * 8192
    need = 2 * (M * 128 * 4 + M * 512 * 2) + (2 * 128 + 512) * 2048 * 2
    assert need <= extra <= need + 8 * 1024 * 1024     # + one GemmSched and alignment
    arr = (C.c_uint64 * 7)()
    for kw in (dict(E=16), dict(dtype="fp32"), dict(k=9)):
        c = dict(G=2, E=32, k=4, H=256, F=256, T=64, h=64, fuse_gate_predictor=True)
        c.update(kw)
        bad = ProbeConfig(**c).to_c()
        assert lib.probe_init(C.byref(bad), arr, C.c_void_p(1024), C.byref(C.c_void_p())) == 2, kw
        assert b"fuse_gate_predictor" in lib.probe_last_error(None)
    assert lib.probe_predict_prepare(None, 1, C.c_void_p(256), None) == 1


def test_fp32_workspace(lib):
    """dtype = PROBE_FP32 (parity path): receive rows, Y and replica slots are fp32, and
    𝒲 = 3·H·F·4 is the checked expert size."""
    from paper_2602_00509_b200 import ProbeConfig, workspace_sizes
    c16 = ProbeConfig(G=2, E=8, k=2, H=256, F=512, T=64, h=64)
    c32 = ProbeConfig(G=2, E=8, k=2, H=256, F=512, T=64, h=64, dtype="fp32")
    s16, s32 = workspace_sizes(c16), workspace_sizes(c32)
    assert c32.to_c().dtype == 1 and c32.expert_bytes == 12 * 256 * 512
    for b in (_lib.BUF_RECV, _lib.BUF_Y, _lib.BUF_REP_W13, _lib.BUF_REP_W2):
        assert s32[b] == 2 * s16[b], b
    assert s32[_lib.BUF_SCRATCH] > s16[_lib.BUF_SCRATCH]
    bad = c32.to_c()
    bad.expert_bytes = 6 * 256 * 512          # the bf16 size is wrong for fp32
    arr = (C.c_uint64 * 7)()
    assert lib.probe_init(C.byref(bad), arr, C.c_void_p(1024), C.byref(C.c_void_p())) == 1
    assert b"sizeof(dtype)" in lib.probe_last_error(None)


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump missing")
def test_sass_is_blackwell_native(lib):
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA tensor loads
    assert "LDTM" in sass             # tcgen05.ld (TMEM → registers)
    assert "HMMA" not in sass.replace("UTCHMMA", "")   # no legacy mma.sync path
