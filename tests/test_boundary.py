"""C-ABI boundary on CPU: libcdsp.so loads and exports every symbol include/cdsp.h declares;
the host-only plan calls agree bit-exactly with the oracle.  No CUDA compute calls."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_2511_06247_b200 import api
from paper_2511_06247_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return api.lib()


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "cdsp.h")).read()
    return sorted(set(re.findall(r"CDSP_API\s+[\w\s\*]+?\b(cdsp_\w+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = _declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), f"libcdsp.so does not export {n}"
    assert set(names) == set(api.EXPORTED_SYMBOLS)
    assert api.abi_version() == 5


def test_no_oracle_in_product():
    """The product path never references the oracle (it shares no code with it)."""
    pkg = os.path.join(ROOT, "paper_2511_06247_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
                assert "oracle_" not in txt, f


PLANS = [
    [(1024, [0, 1])],
    [(512, [0]), (512, [0, 1])],
    [(256, [0, 1]), (256, [0, 1]), (512, [0, 1])],
    [(32768, [0, 1]), (32768, [0, 1, 2, 3]), (32768, list(range(8))), (32768, list(range(8)))],
    [(16384, [0, 1]), (24576, [0, 1, 2, 3]), (40960, list(range(8))), (49152, list(range(8)))],
    [(65536, [0, 1]), (65536, [0, 1, 2, 3]), (131072, list(range(8)))],
    [(64, [3]), (64, [3, 0]), (128, [3, 0, 5, 1]), (96, [3, 0, 5, 1, 2, 4, 6, 7])],
    [(4096, [0, 1, 2, 3]), (4096, list(range(8)))],
]


@pytest.mark.parametrize("plan", PLANS)
def test_plan_partition_matches_oracle(lib, plan):
    P = api.Plan(plan)
    C = 0
    for c, (L, ranks) in enumerate(plan):
        s = len(ranks)
        tr, ts, rp, moves = api.plan_partition(P, c)
        otr, ots = oracle.zigzag_map(L, s)
        np.testing.assert_array_equal(tr, otr)
        np.testing.assert_array_equal(ts, ots)
        np.testing.assert_array_equal(rp, oracle.rank_positions(L, s, C))
        _, _, omoves = oracle.plan_stores(plan, c)
        assert sorted(moves) == sorted(omoves)
        C += L


STRIPED_PLANS = [
    [(1024, [0, 1], "striped")],
    [(512, [0]), (512, [0, 1], "striped"), (1024, [0, 1, 2, 3])],
    [(256, [0, 1], "striped"), (512, [0, 1, 2, 3], "striped"), (1024, list(range(8)), "striped")],
    [(64, [3]), (64, [3, 0], "striped"), (128, [3, 0, 5, 1]), (96, [3, 0, 5, 1, 2, 4, 6, 7], "striped")],
]


@pytest.mark.parametrize("plan", STRIPED_PLANS)
def test_striped_plan_partition_matches_oracle(lib, plan):
    """Chunks interleaved by stripes (R20): maps and shard positions bit-exact vs the oracle;
    balancing moves and store capacity unchanged by the interleave."""
    P = api.Plan(plan)
    C = 0
    for c, chunk in enumerate(plan):
        L, ranks = chunk[0], chunk[1]
        il = chunk[2] if len(chunk) > 2 else "zigzag"
        s = len(ranks)
        tr, ts, rp, moves = api.plan_partition(P, c)
        otr, ots = (oracle.striped_map if il == "striped" else oracle.zigzag_map)(L, s)
        np.testing.assert_array_equal(tr, otr)
        np.testing.assert_array_equal(ts, ots)
        np.testing.assert_array_equal(rp, oracle.rank_positions(L, s, C, interleave=il))
        _, _, omoves = oracle.plan_stores(plan, c)
        assert sorted(moves) == sorted(omoves)
        C += L
    need = 0
    for c, chunk in enumerate(plan):
        n, _, _ = oracle.plan_stores(plan, c)
        need = max(need, int(n.max()) + chunk[0] // len(chunk[1]))
    assert api.plan_capacity(P) == need


@pytest.mark.parametrize("plan", PLANS)
def test_plan_capacity_matches_oracle_stores(lib, plan):
    need = 0
    for c, (L, ranks) in enumerate(plan):
        n, _, _ = oracle.plan_stores(plan, c)
        need = max(need, int(n.max()) + L // len(ranks))
    assert api.plan_capacity(api.Plan(plan)) == need


def test_random_plans_match_oracle(lib):
    rng = np.random.default_rng(5)
    for _ in range(300):
        n_chunks = int(rng.integers(1, 5))
        plan, grp, s = [], [], 1
        pool = list(rng.permutation(8))
        for _ in range(n_chunks):
            s = int(max(s, rng.choice([1, 2, 4, 8])))
            while len(grp) < s:
                grp.append(int(pool.pop()))
            plan.append((2 * s * int(rng.integers(1, 9)), list(grp)))
        P = api.Plan(plan)
        for c in range(len(plan)):
            _, _, _, moves = api.plan_partition(P, c)
            assert sorted(moves) == sorted(oracle.plan_stores(plan, c)[2])


@pytest.mark.parametrize("plan", [
    [(16, [0, 1]), (16, [0])],
    [(16, [0, 1]), (16, [1, 0, 2, 3])],
    [(12, [0, 1, 2])],
    [(18, [0, 1, 2, 3])],
    [(16, [0, 0])],
    [(16, [0, 1]), (24, [0, 1, 2, 3, 4, 5])],
])
def test_illegal_plans_rejected_like_oracle(lib, plan):
    with pytest.raises(oracle.OracleError):
        oracle.plan_stores(plan, len(plan) - 1)
    with pytest.raises(api.CdspError) as e:
        api.plan_partition(api.Plan(plan), len(plan) - 1)
    assert e.value.status == 4  # CDSP_ERR_PLAN
    assert "chunk" in str(e.value)


def test_bad_chunk_index(lib):
    with pytest.raises(api.CdspError) as e:
        api.plan_partition(api.Plan([(16, [0, 1])]), 3)
    assert e.value.status == 1
