"""CDSP prefill scheduler oracle (test infrastructure; only tests/ may import it).

A plain, slow, obviously-correct Python transcription of PAPER.md §5.1 — Eq. (1),
Algorithm 1, Algorithm 2, the instance-group extension,
Algorithm 3 and the queue update Eq. (2) — in the paper's order and
notation.  The readings it takes where the text is silent or garbled are listed in DESIGN.md
(R21-R27) and restated at each step.  The C++ planner in the product (cdsp_schedule_prefill)
shares no code with this module; tests compare the two plan for plan.

Pins (tests/test_planner.py): Eq. (1) recovered exactly from noise-free samples and equal to
numpy.linalg.lstsq on noisy ones; every plan legal (R9) and covering L; the reported TTFT equal
to an independent discrete-event replay of the plan (`replay_ttft`); the P:273 budget example;
single-chunk choice equal to brute force over s under the improvement-rate rule.
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence, Tuple

import numpy as np


# ---- Eq. (1): T_s(R) = a_s + b_s L + c_s (C L) + d_s L^2 ------------------------------
def perf_model(coef: Tuple[float, float, float, float], C: float, L: float) -> float:
    a, b, c, d = coef
    return a + b * L + c * (C * L) + d * L * L


def fit_model(C: Sequence[float], L: Sequence[float], T: Sequence[float]):
    """Least-squares fit of Eq. (1) ("obtained from least-squares fitting by collecting
    latency data across various (C, L) pairs"): the library routine is the step."""
    C, L, T = (np.asarray(x, np.float64) for x in (C, L, T))
    X = np.stack([np.ones_like(L), L, C * L, L * L], axis=1)
    return tuple(float(x) for x in np.linalg.lstsq(X, T, rcond=None)[0])


# ---- instance-group extension (GetGroup) -----------------------------------------------
# The pool P is a dict instance id -> queuing latency T_i; instance i sits on node
# i // node_size (nodes of consecutive ids).  Ties break by lower id / lower node (R22).
def _node_of(i: int, node_size: int) -> int:
    return i // node_size


def _shortest(ids, pool, n: int) -> List[int]:
    return sorted(ids, key=lambda i: (pool[i], i))[:n]


def get_group(pool: Dict[int, float], node_size: int, initial: List[int], s: int):
    """Extend `initial` (its ring order kept, R9) to s instances of the pool, or None (R23)."""
    if s < len(initial) or s > len(pool):
        return None
    group = list(initial)
    used = set(group)
    need = s - len(group)
    if need == 0:
        return group
    # (2) "first adds instances within the nodes containing initial_group's instances"
    if group:
        home = {_node_of(i, node_size) for i in group}
        cand = [i for i in pool if _node_of(i, node_size) in home and i not in used]
        for i in _shortest(cand, pool, need):
            group.append(i)
            used.add(i)
        need = s - len(group)
        if need == 0:
            return group
    # (1) on the remaining free nodes
    members: Dict[int, List[int]] = {}
    for i in pool:
        members.setdefault(_node_of(i, node_size), []).append(i)
    free_nodes = sorted(nd for nd, mem in members.items() if not any(i in used for i in mem))
    k_full = need // node_size
    if k_full > 0:
        # "if s spans k full nodes, the algorithm selects the top-k nodes with the shortest
        # queuing latency" — a node's latency = its longest queue (R22); full nodes only
        full = [nd for nd in free_nodes if len(members[nd]) == node_size]
        order = sorted(full, key=lambda nd: (max(pool[i] for i in members[nd]), nd))
        if len(order) < k_full:
            return None
        for nd in order[:k_full]:
            for i in _shortest(members[nd], pool, node_size):
                group.append(i)
                used.add(i)
            free_nodes.remove(nd)
        need = s - len(group)
    if need > 0:
        # "selects the node with the minimal s-th shortest queuing latency and takes its s
        # shortest-queued instances"
        best = None
        for nd in free_nodes:
            if len(members[nd]) < need:
                continue
            key = (sorted(pool[i] for i in members[nd])[need - 1], nd)
            if best is None or key < best:
                best = key
        if best is None:
            return None
        for i in _shortest(members[best[1]], pool, need):
            group.append(i)
            used.add(i)
    return group


# ---- Algorithm 2: single-chunk scheduling ------------------------------------------------------
def single_chunk_schedule(L: int, A: list, S: Sequence[int], pool: Dict[int, float], node_size: int,
                          models: Dict[int, tuple], rate: float):
    C = sum(c[0] for c in A)                          # line 4
    initial = list(A[-1][1]) if A else []             # line 5: all instances of A (last group, R9)
    opt_ttft, opt_group, opt_s = math.inf, None, None
    for s in sorted(S):                               # line 6
        group = get_group(pool, node_size, initial, s)    # line 8
        if group is None:
            continue
        t_queue = max(pool[i] for i in group)         # line 9
        t_prefill = perf_model(models[s], C, L)       # line 10
        ttft = t_queue + t_prefill                    # line 11
        if ttft < opt_ttft * (1.0 - rate):            # line 13 (INF * x = INF: first s taken)
            opt_ttft, opt_group, opt_s = ttft, group, s
    return opt_group, opt_ttft


# ---- Algorithm 3: chunk plan solving ----------------------------------------------------------
def solve_chunk_len(coef, C: float, budget: float) -> float:
    """Largest L with Eq. (1) <= budget (a polynomial in the chunk size, solved
    numerically): d L^2 + (b + c C) L + (a - budget) = 0, positive root (R24)."""
    a, b, c, d = coef
    B = b + c * C
    if budget <= a:
        return 0.0
    if d <= 0.0:
        return (budget - a) / B if B > 0 else math.inf
    return (-B + math.sqrt(B * B + 4.0 * d * (budget - a))) / (2.0 * d)


def chunk_plan_solve(L: int, A: list, s_cur: int, s_next: int, pool, node_size, models, granule):
    C = sum(c[0] for c in A)                                           # line 3
    initial = list(A[-1][1]) if A else []                              # line 4
    cur = get_group(pool, node_size, initial, s_cur)                   # line 6
    if cur is None:
        return None
    nxt = get_group(pool, node_size, cur, s_next)                      # line 7
    if nxt is None:
        return None
    t_cur = max(pool[i] for i in cur)                                  # line 9
    t_next = max(pool[i] for i in nxt)                                 # line 10
    budget = t_next - t_cur                                            # line 11
    l_chunk = min(L, solve_chunk_len(models[s_cur], C, budget))        # line 13
    l_chunk = int(l_chunk // granule) * granule                        # R25: whole granules (exact floor)
    return l_chunk, cur


def illegal(l_chunk: int, L: int) -> bool:
    """R26: "negative chunk sizes or chunk lengths that are too short to yield benefits"."""
    return l_chunk <= 0 or l_chunk >= L


# ---- Algorithm 1: CDSP scheduling -------------------------------------------------------------
def cdsp_schedule(L: int, A: list, S: Sequence[int], pool: Dict[int, float], node_size: int,
                  models: Dict[int, tuple], rate: float, granule: int):
    """-> (allocation [(len, ring-order group)], TTFT relative to now).  The paper's line 11
    reads "if Illegal(...)": the recursion runs for LEGAL plans (R27)."""
    group, ttft = single_chunk_schedule(L, A, S, pool, node_size, models, rate)    # line 3
    if group is None:
        return None, math.inf
    opt = (A + [(L, group)], ttft)                                                 # line 4
    s_cdsp = [s for s in S if s <= len(group)]                                     # line 6
    pairs = [(a, b) for a in sorted(s_cdsp) for b in sorted(s_cdsp) if a < b]      # line 7
    in_group = {i: pool[i] for i in group}  # line 10 solves within instance_group, not all of P
    for s_cur, s_next in pairs:                                                    # line 8
        plan = chunk_plan_solve(L, A, s_cur, s_next, in_group, node_size, models, granule)  # line 10
        if plan is None or illegal(plan[0], L):                                    # line 11 (R27)
            continue
        l_chunk, cur = plan
        C = sum(c[0] for c in A)
        t_queue = max(in_group[i] for i in cur)
        t_prefill = perf_model(models[s_cur], C, l_chunk)
        elapsed = t_queue + t_prefill
        # line 16, Eq. (2): P' = instance_group with T_i <- max{0, T_i - (T_queue + T_prefill)} (R21)
        pool2 = {i: max(0.0, pool[i] - elapsed) for i in group}
        S2 = [s for s in s_cdsp if s >= s_next]                                    # line 15
        alloc, rest = cdsp_schedule(L - l_chunk, A + [(l_chunk, cur)], S2, pool2, node_size, models, rate,
                                    granule)                                       # lines 13-17
        if alloc is None:
            continue
        if elapsed + rest < opt[1]:                                                # line 19
            opt = (alloc, elapsed + rest)                                          # line 20
    return opt


# ---- independent replay (a pin for the TTFT arithmetic) --------------------------------------
def replay_ttft(alloc, queue: Dict[int, float], models) -> float:
    """Discrete-event replay: chunk i starts when its whole group is free and chunk i-1 has
    finished ("All instance groups compute sequentially following the chunk order")."""
    t, C = 0.0, 0
    for L, grp in alloc:
        start = max([t] + [queue[i] for i in grp])
        t = start + perf_model(models[len(grp)], C, L)
        C += L
    return t
