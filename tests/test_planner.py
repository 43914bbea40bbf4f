"""CPU: the CDSP prefill scheduler (§5.1, Eq. 1, Alg. 1-3).

Oracle pins (oracle/planner.py against the paper and arithmetic, not against itself), then
parity of the product's C++ planner (cdsp_schedule_prefill, cdsp_fit_latency_model) with the
oracle, plan for plan, and its latency against Table 2."""
import math
import time

import numpy as np
import pytest

import oracle
from oracle import planner as P

S = [1, 2, 4, 8]


def _models(rng):
    """Eq. (1) coefficients shaped like prefill (ms; C, L in tokens): constant, FC-linear,
    history-attention and within-chunk-attention terms, each shrinking with s."""
    m = {}
    for s in S:
        f = 1.0 / s ** rng.uniform(0.8, 1.0)
        m[s] = (rng.uniform(0.5, 3.0) * (1 + 0.1 * s), rng.uniform(1e-4, 4e-4) * f,
                rng.uniform(1e-9, 4e-9) * f, rng.uniform(0.5e-9, 2e-9) * f)
    return m


def _case(rng):
    n_inst = int(rng.choice([8, 16, 24]))
    q = rng.exponential(rng.uniform(10, 400), n_inst) * (rng.random(n_inst) < 0.7)
    queue = {i: float(q[i]) for i in range(n_inst)}
    granule = 2 * 8 * int(rng.choice([64, 128]))
    L = granule * int(rng.integers(1, 64))
    return L, queue, 8, _models(rng), float(rng.choice([0.0, 0.05, 0.1, 0.3, 0.5])), granule


# ---- oracle pins -----------------------------------------------------------------------------
def test_fit_recovers_eq1_exactly():
    rng = np.random.default_rng(0)
    truth = (1.5, 2e-4, 3e-9, 1e-9)
    C = rng.integers(0, 200000, 64).astype(float)
    L = rng.integers(1024, 200000, 64).astype(float)
    T = [P.perf_model(truth, c, l) for c, l in zip(C, L)]
    fit = P.fit_model(C, L, T)
    for a, b in zip(fit, truth):
        assert abs(a - b) <= 1e-6 * abs(b) + 1e-12


def test_plans_legal_cover_prompt_and_ttft_replays():
    rng = np.random.default_rng(1)
    n_multi = 0
    for _ in range(300):
        L, queue, node, models, rate, granule = _case(rng)
        alloc, ttft = P.cdsp_schedule(L, [], S, queue, node, models, rate, granule)
        assert alloc is not None
        assert sum(c[0] for c in alloc) == L
        assert all(c[0] % granule == 0 for c in alloc[:-1])
        oracle.plan_stores([(c[0], c[1]) for c in alloc], len(alloc) - 1)  # raises on an illegal plan (R9)
        assert math.isclose(ttft, P.replay_ttft(alloc, queue, models), rel_tol=1e-12, abs_tol=1e-9)
        n_multi += len(alloc) > 1
    assert n_multi >= 10  # chunking happens under queueing


def test_budget_example_p273():
    """"when solving the plan for chunk 1 with s_current=2 and s_next=4, the budget is
    obtained by comparing the maximum queuing latencies of instances 0-3 and 2-3"."""
    queue = dict(enumerate([50.0, 40.0, 5.0, 10.0, 90.0, 90.0, 90.0, 90.0]))
    m = {2: (0.0, 1e-3, 0.0, 0.0), 4: (0.0, 5e-4, 0.0, 0.0)}
    l_chunk, cur = P.chunk_plan_solve(10 ** 9, [], 2, 4, queue, 4, m, 1)
    assert sorted(cur) == [2, 3]
    budget = max(queue[i] for i in range(4)) - max(queue[2], queue[3])
    assert l_chunk == int(budget / 1e-3)


def test_no_queueing_means_single_chunk_at_argmin():
    rng = np.random.default_rng(3)
    for _ in range(50):
        models = _models(rng)
        L = 1024 * int(rng.integers(1, 128))
        alloc, ttft = P.cdsp_schedule(L, [], S, dict.fromkeys(range(16), 0.0), 8, models, 0.0, 1024)
        assert len(alloc) == 1
        best = min(P.perf_model(models[s], 0, L) for s in S)
        assert math.isclose(ttft, best, rel_tol=1e-12)


def test_improvement_rate_limits_expansion():
    """Alg. 2 line 13: a larger SP is taken only if it improves TTFT by more than the rate."""
    models = {s: (0.0, 1.0 / s ** 0.3, 0.0, 0.0) for s in S}  # weak scaling: 2^-0.3 = 0.81 per doubling
    free = dict.fromkeys(range(8), 0.0)
    g0, _ = P.single_chunk_schedule(1000, [], S, free, 8, models, 0.0)
    g1, _ = P.single_chunk_schedule(1000, [], S, free, 8, models, 0.25)
    g2, _ = P.single_chunk_schedule(1000, [], S, free, 8, models, 0.6)
    # rate 0.25: s=2 (812) misses 0.75 x 1000, s=4 (660) makes it, s=8 (536) misses 0.75 x 660
    assert len(g0) == 8 and len(g1) == 4 and len(g2) == 1


def test_get_group_prefers_one_node_and_extends_home_nodes():
    queue = dict(enumerate([9, 9, 9, 9, 1, 2, 3, 30] + [0, 0, 50, 50, 50, 50, 50, 50]))
    g = P.get_group(queue, 8, [], 2)
    assert sorted(g) == [8, 9]                     # node 1's 2nd-shortest queue (0) beats node 0's (2)
    g = P.get_group(queue, 8, [8, 9], 4)
    assert g[:2] == [8, 9] and all(i >= 8 for i in g)  # extended inside the home node first
    g = P.get_group(queue, 8, [], 16)
    assert sorted(g) == list(range(16))


# ---- product parity (C++ planner vs the oracle) ----------------------------------------------
def _lib():
    from paper_2511_06247_b200 import api
    from paper_2511_06247_b200.build import build
    build()
    return api


def test_cpp_fit_matches_oracle():
    api = _lib()
    rng = np.random.default_rng(7)
    for _ in range(20):
        truth = (rng.uniform(0, 5), rng.uniform(1e-5, 1e-3), rng.uniform(1e-10, 1e-8), rng.uniform(1e-10, 1e-8))
        C = rng.integers(0, 300000, 40).astype(float)
        L = rng.integers(1024, 200000, 40).astype(float)
        T = np.array([P.perf_model(truth, c, l) for c, l in zip(C, L)]) * rng.normal(1, 0.02, 40)
        mine, ref = api.fit_latency_model(C, L, T), P.fit_model(C, L, T)
        for a, b in zip(mine, ref):
            assert abs(a - b) <= 1e-6 * max(abs(b), 1e-12) + 1e-9 * abs(truth[0])
        # noise-free: exact recovery
        T0 = [P.perf_model(truth, c, l) for c, l in zip(C, L)]
        for a, b in zip(api.fit_latency_model(C, L, T0), truth):
            assert abs(a - b) <= 1e-6 * abs(b)


def test_cpp_planner_matches_oracle_plan_for_plan():
    api = _lib()
    rng = np.random.default_rng(11)
    n_multi = 0
    for _ in range(400):
        L, queue, node, models, rate, granule = _case(rng)
        ref, ref_ttft = P.cdsp_schedule(L, [], S, queue, node, models, rate, granule)
        plan, ttft = api.schedule_prefill(L, [queue[i] for i in range(len(queue))], node, models, rate, granule)
        assert plan == [(c[0], list(c[1])) for c in ref]
        assert abs(ttft - ref_ttft) <= 1e-12 * abs(ref_ttft)  # plans exact; TTFT to rounding order
        n_multi += len(plan) > 1
        api.plan_partition(api.Plan(plan), len(plan) - 1)  # the library accepts its own plans
    assert n_multi >= 5


def test_cpp_planner_latency_vs_table2():
    """Table 2: <= 86.8 us per scheduling call on the authors' host; measured here on
    this host's CPU for pools of 8-32 instances (our plans cap SP at 8)."""
    api = _lib()
    rng = np.random.default_rng(13)
    cases = [_case(rng) for _ in range(200)]
    t0 = time.perf_counter()
    for L, queue, node, models, rate, granule in cases:
        api.schedule_prefill(L, [queue[i] for i in range(len(queue))], node, models, rate, granule)
    per_call_us = (time.perf_counter() - t0) / len(cases) * 1e6
    assert per_call_us < 2000  # includes ctypes marshalling; the C++ call alone is reported in DESIGN
