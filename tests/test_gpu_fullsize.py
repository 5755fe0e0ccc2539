"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(8 logical EP ranks on one B200, capacity 4·T·k, planner constants from measured peaks).

Routing, counts, predicted counts, plan, split, dispatch route and group sizes are
compared bit-exactly over ALL tokens; layer outputs on a per-rank token sample
(always including the last, ragged-tail token) within 2e-2·RMS.
"""
import pytest

import probe_inputs as pi
from layer_harness import CaseCfg, compare, run_gpu, run_oracle
from paper_2602_00509_b200.costs import cost_model, window_ns

pytestmark = pytest.mark.gpu


def bench_case(shape, zipf_s=1.0, sample=24, cap=4.0):
    a, b, n, bw = cost_model(shape.H, shape.F)
    return CaseCfg(shape, zipf_s=zipf_s, alpha_ps=a, beta_ps=b, n_sat=n, bw_bytes_per_us=bw,
                   window_ns=window_ns(shape.H, shape.F, shape.T, shape.k, E=shape.E, G=shape.G), capacity_factor=cap,
                   sample_tokens=sample)


@pytest.mark.parametrize("name,case", [
    ("C1-bench", bench_case(pi.C1)),
    ("C1-s1.5", bench_case(pi.C1, zipf_s=1.5)),
    ("C2-decode", bench_case(pi.C2, sample=32)),
    ("C3-T2048", bench_case(pi.C3.with_(T=2048), sample=8, cap=3.0)),
])
def test_fullsize_parity(name, case):
    gpu, inputs = run_gpu(case)
    orc = run_oracle(case, inputs)
    rep = compare(case, gpu, orc, tol=2e-2)
    print(name, rep)
