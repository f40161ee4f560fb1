"""Host-side planner checks (no GPU): the recursion shapes the scheduler
(step a6) builds for every BASELINE config, through the C ABI's
toom_plan_describe.  The shapes follow SURVEY.md §8(d) / DESIGN.md §2
reading 8: Toom-4 while n > t4, Toom-3 while n > t3, schoolbook below; 2B-1
children per parent; evaluated widths e = b + growth limbs."""
import math

import pytest

import paper_1602_02740_b200 as tg


def levels(n, batch, B, **kw):
    return tg.plan_describe(n, batch, B=B, **kw)["levels"]


def check_counts(lv, batch):
    assert lv[0]["count"] == batch
    for a, b in zip(lv, lv[1:]):
        assert b["count"] == a["count"] * a["npts"]
        assert a["npts"] == 2 * a["B"] - 1
        assert b["n"] == a["e"]
        assert a["b"] == math.ceil(a["n"] / a["B"])
        assert a["lentop"] == a["n"] - (a["B"] - 1) * a["b"] and a["lentop"] >= 1
        assert a["Lw"] == 2 * a["b"] + 1


def test_c1_plan():
    lv = levels(96, 260, 3, t4=10**9, t3=10**9)
    check_counts(lv, 260)
    assert [L["B"] for L in lv] == [3, 0] and lv[0]["e"] == 33 and lv[1]["n"] == 33


def test_c2_plan():
    info = tg.plan_describe(256, 65536, B=4, t4=32, t3=32)
    lv = info["levels"]
    check_counts(lv, 65536)
    assert [L["B"] for L in lv] == [4, 4, 0]
    assert [L["n"] for L in lv] == [256, 65, 18]          # "recursing to a 32-limb schoolbook base"
    assert info["fused_bottom"] and not any(L["long"] for L in lv)


def test_c3_plan():
    lv = levels(2048, 4096, 8)
    check_counts(lv, 4096)
    assert [L["B"] for L in lv] == [8, 4, 3, 0]
    assert [L["n"] for L in lv] == [2048, 258, 66, 23]   # Toom-8 (paper points) -> Toom-4/3 -> schoolbook <= 64


def test_c4_plan():
    info = tg.plan_describe(1 << 20, 1, B=4)
    lv = info["levels"]
    check_counts(lv, 1)
    assert lv[-1]["B"] == 0 and lv[-1]["n"] <= 64
    assert all(L["B"] in (3, 4) for L in lv[:-1])
    # few long operands at the top run limb-parallel, the rest instance-parallel
    assert lv[0]["long"] and not lv[-2]["long"] and info["fused_bottom"]
    longs = [L["long"] for L in lv[:-1]]
    assert longs == sorted(longs, reverse=True)             # a prefix


def test_c5_plan():
    info = tg.plan_describe(1 << 24, 1, B=16)
    lv = info["levels"]
    check_counts(lv, 1)
    assert lv[0]["B"] == 16 and lv[0]["npts"] == 31 and lv[0]["long"]
    assert lv[0]["b"] == 1 << 20 and lv[0]["e"] == (1 << 20) + 2   # 35.6 bits of growth -> 2 limbs
    assert lv[1]["count"] == 31


@pytest.mark.parametrize("B", [3, 4, 8, 16])
def test_eval_width_growth(B):
    # e - b limbs hold the growth of the largest point value sum_k |p^k q^(n-k)|
    growth = {3: 1, 4: 1, 8: 2, 16: 2}[B]
    n = 1000 * B
    assert tg.lib().toom_eval_width(n, B) == math.ceil(n / B) + growth
    assert tg.lib().toom_npoints(B) == 2 * B - 1


def test_long_count_controls():
    never = levels(1 << 20, 1, 4, long_count=1)
    assert not any(L["long"] for L in never[:-1] if L["B"] != 16)
    always = levels(300, 9, 3, long_count=1 << 30)
    # every Toom level above the fused bottom level is long (the lazy block,
    # csrc/lazy.cuh, ends at the fused level, which stays instance-parallel)
    assert all(L["long"] for L in always[:-2])
    assert always[0]["lazy"] and not always[-2]["long"]


def test_workspace_grows_with_batch():
    a = tg.workspace_bytes(256, 1024, B=4, t4=32, t3=32)
    b = tg.workspace_bytes(256, 4096, B=4, t4=32, t3=32)
    assert 0 < a < b


def test_c2_plan_uses_the_common_denominator_kernels():
    """C2 (BASELINE configs[1]): c2 mode 2 (deferred bottom + top by classes,
    DESIGN.md reading 18); other shapes keep the per-row kernels."""
    assert tg.plan_describe(256, 65536, B=4, t4=32, t3=32)["c2_mode"] == 2
    assert tg.plan_describe(256, 1000, B=4, t4=32, t3=32)["c2_mode"] == 2
    assert tg.plan_describe(96, 260, B=3, t4=10**9, t3=10**9)["c2_mode"] == 0
    assert tg.plan_describe(2048, 4096, B=8)["c2_mode"] == 0
    tg.set_c2_mode(0)
    try:
        assert tg.plan_describe(256, 65536, B=4, t4=32, t3=32)["c2_mode"] == 0
    finally:
        tg.set_c2_mode(2)
