"""Values outside the packed / 16-bit forms: the reference computes the bound in plain
int (bound.hpp:27-44, 61-90); the device path must give the same bounds for every
instance fbb_create accepts (total processing time <= 2^30, n <= 256, m <= 64).

build_host_tables (csrc/tables.cu) bounds every max-plus intermediate per instance and
picks the kernels whose 16-bit arithmetic is exact for it (DevTables::safe16), else the
int32 kWide kernels.  Each case here is checked against the oracle, K1 and K2, and the
kernel choice is asserted so that every form is exercised."""
import numpy as np
import pytest

import paper_1206_4973_b200 as fbb

pytestmark = pytest.mark.gpu


def _check(oracle, p, rng, nodes=200, parents=6, seed_depths=None):
    n, m = p.shape
    inst = fbb.Instance(n, m, p)
    ctx = fbb.Context(inst)
    # K1 on random nodes (all depths, leaves included)
    pre = [list(rng.permutation(n)[: rng.integers(0, n + 1)]) for _ in range(nodes)]
    nb = fbb.nodes_from_prefixes(inst, pre)
    got = ctx.bound(nb)
    ref = oracle.evaluate_batch(p, nb.masks, nb.heads, nb.depth)
    assert np.array_equal(got, ref), "K1"
    # K2: random parents in pop order, frozen at the median child bound, and solve mode
    par = sorted([list(rng.permutation(n)[: rng.integers(0, n)]) for _ in range(parents)],
                 key=len, reverse=True)
    kids = []
    for pr in par:
        kids += oracle.branch(p, pr)[0]
    kn = fbb.nodes_from_prefixes(inst, kids)
    klb = oracle.evaluate_batch(p, kn.masks, kn.heads, kn.depth)
    for frozen in (True, False):
        ub = int(np.percentile(klb, 50)) + 1
        leaf = [int(v) for k, v in zip(kids, klb) if len(k) == n]
        inc = ub if frozen else min([ub] + leaf)
        surv, slb, *_ = ctx.expand_bound_prune(fbb.nodes_from_prefixes(inst, par), ub, frozen)
        exp = [(k, int(v)) for k, v in zip(kids, klb) if len(k) < n and v < inc]
        assert surv.prefixes() == [k for k, _ in exp], f"K2 frozen={frozen}"
        assert list(slb) == [v for _, v in exp], f"K2 bounds frozen={frozen}"
    return ctx.kernels()


def test_int16_overflow_cases_from_review(oracle):
    rng = np.random.default_rng(1)
    # n=20, m=20, p[j][0]=982, p[j][1..19]=855: |d| <= 127 (register-row tables), but
    # Lc_1 + M'_01 reaches 34,903 -- the 16x2 Phase B would wrap
    p = np.full((20, 20), 855, np.int32)
    p[:, 0] = 982
    k = _check(oracle, p, rng, nodes=300, parents=12)
    assert "k2_v2_kernel<20,20,3>" in k, k  # per-pair Phase B (int32 Lc + M')
    # the same shape with noise
    p2 = p + rng.integers(-5, 6, size=p.shape).astype(np.int32)
    _check(oracle, p2, rng, nodes=300, parents=12)
    # n=200, m=2, p=[290, 40]: d = 250 (generic kernel), M' reaches 49,790
    p = np.tile(np.array([290, 40], np.int32), (200, 1))
    k = _check(oracle, p, rng, nodes=120, parents=6)
    assert "k2_internal_kernel<0,1>" in k, k
    # n=200, m=3, p=(255,1,1) (the advisor's case)
    p = np.tile(np.array([255, 1, 1], np.int32), (200, 1))
    k = _check(oracle, p, rng, nodes=120, parents=6)
    assert "k2_internal_kernel<0,1>" in k and "k1_bound_kernel" in k, k


@pytest.mark.parametrize("m", [2, 3, 20])
def test_random_p_up_to_255_at_n200(oracle, m):
    rng = np.random.default_rng(100 + m)
    p = rng.integers(1, 256, size=(200, m)).astype(np.int32)
    _check(oracle, p, rng, nodes=80 if m == 20 else 200, parents=4 if m == 20 else 8)


def test_random_p_850_980_at_20x20(oracle):
    rng = np.random.default_rng(7)
    for trial in range(3):
        p = rng.integers(850, 981, size=(20, 20)).astype(np.int32)
        _check(oracle, p, rng, nodes=300, parents=16)


def test_unpacked_values_run_the_wide_kernels(oracle):
    # |p[j][k] - p[j][l]| > 255 and c = sum of a pair span >= 2^14: no packed table at all
    rng = np.random.default_rng(9)
    for (n, m, hi) in [(12, 4, 5000), (30, 6, 3000), (70, 3, 20000), (20, 20, 2000)]:
        p = rng.integers(1, hi, size=(n, m)).astype(np.int32)
        k = _check(oracle, p, rng, nodes=200, parents=8)
        assert "k1_bound_kernel<0,0,1>" in k and "k2_internal_kernel<0,1>" in k, k


def test_explorer_with_wide_values_matches_reference(oracle):
    # a whole frozen exploration and a solve on an instance outside the packed range
    rng = np.random.default_rng(21)
    p = rng.integers(1, 3000, size=(9, 4)).astype(np.int32)
    inst = fbb.Instance(9, 4, p)
    opt, sched, _ = oracle.solve(p, -1, targets=[64])
    res, gold = oracle.resolve(p, opt["optimum"] + 50, [[]], targets=[32], max_trace=4096)
    got = fbb.resolve_workload(inst, [[]], opt["optimum"] + 50, targets=[32])
    assert [tuple(r) for r in got.rounds] == [tuple(r) for r in gold]
    sol = fbb.solve(inst, targets=[32])
    assert sol.optimum == opt["optimum"]
    assert fbb.makespan(inst, sol.schedule) == opt["optimum"]


def test_total_beyond_int32_is_rejected():
    p = np.full((64, 64), 300_000, np.int32)  # sum = 1.2e9 > 2^30
    with pytest.raises(fbb.BackendError) as e:
        fbb.Context(fbb.Instance(64, 64, p))
    assert e.value.status == fbb._lib.FBB_E_RANGE
