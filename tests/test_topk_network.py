"""CPU check of the sorting networks the top-k select kernel and the GEMM-epilogue top-k use
(gemm_sm100.cuh topk_sort8 / topk_merge8).  The comparator lists are parsed from the CUDA source and simulated here:
by the 0-1 principle, a comparator network sorts every input iff it sorts every 0-1 input,
so sort8 is checked on all 2^8 binary vectors, and the merge (element-wise better of
top[i] and group[7-i], then the bitonic cleaner) on all pairs of sorted binary lists; plus
random (value, id) keys with heavy ties against Python's sort by (value ↓, id ↑) (R3, R4)."""
import itertools
import os
import random
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "paper_2602_00509_b200", "csrc", "gemm_sm100.cuh")).read()


def _pairs(fn):
    body = SRC[SRC.index(f"void {fn}("):]
    body = body[:body.index("#undef CE")]
    return [(int(a), int(b)) for a, b in re.findall(r"CE\((\d+), (\d+)\)", body)]


SORT8 = _pairs("topk_sort8")
CLEAN8 = _pairs("topk_merge8")


def better(a, b):            # key a before key b: value ↓, id ↑
    return a[0] > b[0] or (a[0] == b[0] and a[1] < b[1])


def run(net, xs):
    xs = list(xs)
    for i, j in net:
        if better(xs[j], xs[i]):
            xs[i], xs[j] = xs[j], xs[i]
    return xs


def merge(top, grp):
    c = [grp[7 - i] if better(grp[7 - i], top[i]) else top[i] for i in range(8)]
    return run(CLEAN8, c)


def ref(keys):
    return sorted(keys, key=lambda k: (-k[0], k[1]))


def test_network_shapes():
    assert len(SORT8) == 19 and len(CLEAN8) == 12


def test_sort8_zero_one_principle():
    for bits in itertools.product([0, 1], repeat=8):
        keys = [(b, 0) for b in bits]          # equal ids: values alone must end up sorted
        out = run(SORT8, keys)
        assert [k[0] for k in out] == sorted(bits, reverse=True)


def test_merge_zero_one_principle():
    for a in range(9):
        for b in range(9):
            top = [(1, 0)] * a + [(0, 0)] * (8 - a)
            grp = [(1, 0)] * b + [(0, 0)] * (8 - b)
            out = merge(top, grp)
            assert [k[0] for k in out] == [1] * min(8, a + b) + [0] * (8 - min(8, a + b))


def test_streamed_topk_random_with_ties():
    r = random.Random(5)
    for _ in range(300):
        E = 8 * r.randint(1, 32)
        vals = [r.choice([0.0, 0.5, 1.0, -1.0, 2.0]) if r.random() < 0.5 else r.random() for _ in range(E)]
        keys = list(zip(vals, range(E)))
        top = [(-float("inf"), 0x7fffffff)] * 8
        for g in range(0, E, 8):
            top = merge(top, run(SORT8, keys[g:g + 8]))
        assert top == ref(keys)[:8]
