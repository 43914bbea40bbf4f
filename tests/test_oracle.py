"""Pins for the CPU oracle (oracle/cdsp_oracle.c) against things other than itself:
library routines it reduces to, closed forms, brute force on tiny inputs, invariants the
paper states, and the paper's worked examples (tests/golden/).  CPU only."""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from cdsp_inputs import qkv

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _sdpa_ref(q, k, v, scale):
    """torch SDPA (library, float64, CPU) causal attention + torch.logsumexp of the masked
    scores.  q [N,Hq,D], k/v [N,Hkv,D]."""
    q64 = torch.as_tensor(q, dtype=torch.float64).permute(1, 0, 2)
    k64 = torch.as_tensor(k, dtype=torch.float64).permute(1, 0, 2)
    v64 = torch.as_tensor(v, dtype=torch.float64).permute(1, 0, 2)
    g = q64.shape[0] // k64.shape[0]
    k64 = k64.repeat_interleave(g, 0)
    v64 = v64.repeat_interleave(g, 0)
    o = torch.nn.functional.scaled_dot_product_attention(q64[None], k64[None], v64[None],
                                                         is_causal=True, scale=scale)[0]
    N = q64.shape[1]
    sc = torch.einsum("hqd,hkd->hqk", q64, k64) * scale
    sc = sc.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    return o.permute(1, 0, 2).numpy(), torch.logsumexp(sc, dim=-1).numpy()


@pytest.mark.parametrize("N,Hq,Hkv,D", [(1, 2, 2, 8), (37, 4, 4, 16), (70, 8, 2, 32), (129, 4, 1, 64)])
@pytest.mark.parametrize("sharp", [False, True])
def test_attention_matches_sdpa(N, Hq, Hkv, D, sharp):
    q, k, v = (t.numpy() for t in qkv(N, Hq, Hkv, D, torch.float32, seed=N, sharp=sharp))
    scale = 1.0 / math.sqrt(D)
    out, lse = oracle.causal_rows(q, k, v, scale)
    o_ref, l_ref = _sdpa_ref(q, k, v, scale)
    np.testing.assert_allclose(out, o_ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse, l_ref, rtol=0, atol=1e-12)


def test_attention_row_subset_and_custom_scale():
    N, H, D = 50, 2, 8
    q, k, v = (t.numpy() for t in qkv(N, H, H, D, torch.float32, seed=3))
    rows = np.array([49, 0, 17, 17, 31])
    full_o, full_l = oracle.causal_rows(q, k, v, 0.37)
    o, l = oracle.causal_rows(q, k, v, 0.37, rows=rows)
    np.testing.assert_array_equal(o, full_o[rows])
    np.testing.assert_array_equal(l, full_l[:, rows])
    o_ref, l_ref = _sdpa_ref(q, k, v, 0.37)
    np.testing.assert_allclose(o, o_ref[rows], atol=1e-12, rtol=0)


def test_closed_form_zero_query():
    """q = 0: uniform weights over the visible prefix -> o_t = mean_{j<=t} v_j, lse = ln(t+1)."""
    N, H, D = 33, 2, 4
    _, k, v = (t.numpy() for t in qkv(N, H, H, D, torch.float32, seed=5))
    q = np.zeros((N, H, D), np.float32)
    out, lse = oracle.causal_rows(q, k, v, 0.5)
    csum = np.cumsum(v.astype(np.float64), axis=0) / np.arange(1, N + 1)[:, None, None]
    np.testing.assert_allclose(out, csum, atol=1e-13, rtol=0)
    np.testing.assert_allclose(lse, np.log(np.arange(1, N + 1))[None, :].repeat(H, 0), atol=1e-13, rtol=0)


def test_closed_form_first_token_and_equal_keys():
    N, H, D = 9, 3, 8
    q, k, v = (t.numpy() for t in qkv(N, H, H, D, torch.float32, seed=6))
    out, lse = oracle.causal_rows(q, k, v, 0.25)
    # t = 0 sees only itself: o_0 = v_0 exactly, lse_0 = sigma <q_0, k_0>
    np.testing.assert_array_equal(out[0], v[0].astype(np.float64))
    np.testing.assert_allclose(lse[:, 0], 0.25 * np.einsum("hd,hd->h", q[0].astype(np.float64),
                                                            k[0].astype(np.float64)), atol=1e-14)
    # all keys equal: the scores are equal -> uniform weights, as in the q = 0 case
    k_eq = np.repeat(k[:1], N, axis=0)
    out2, _ = oracle.causal_rows(q, k_eq, v, 0.25)
    np.testing.assert_allclose(out2, np.cumsum(v.astype(np.float64), 0) / np.arange(1, N + 1)[:, None, None],
                               atol=1e-13)


def test_one_hot_values_give_probability_rows():
    """v_j = e_j (N <= D): o_t is the attention probability row; it sums to 1 and is 0
    beyond t (causality), and its log ratios reproduce the score differences."""
    N, H, D = 12, 2, 16
    q, k, _ = (t.numpy() for t in qkv(N, H, H, D, torch.float32, seed=8))
    v = np.zeros((N, H, D), np.float32)
    for j in range(N):
        v[j, :, j] = 1.0
    out, lse = oracle.causal_rows(q, k, v, 0.3)
    for t in range(N):
        p = out[t, :, :N]
        np.testing.assert_allclose(p.sum(-1), 1.0, atol=1e-14)
        assert np.all(p[:, t + 1:] == 0.0)
        s = 0.3 * np.einsum("hd,jhd->hj", q[t].astype(np.float64), k[: t + 1].astype(np.float64))
        np.testing.assert_allclose(np.log(p[:, : t + 1]), s - lse[:, t:t + 1], atol=1e-12)


def test_brute_force_tiny():
    """Explicit enumeration of exp/sum in Python on a 5-token prompt (brute force)."""
    N, H, D = 5, 1, 3
    q, k, v = (t.numpy().astype(np.float64) for t in qkv(N, H, H, D, torch.float32, seed=9))
    out, lse = oracle.causal_rows(q, k, v, 0.7)
    for t in range(N):
        w = [math.exp(0.7 * sum(q[t, 0, d] * k[j, 0, d] for d in range(D))) for j in range(t + 1)]
        Z = sum(w)
        assert abs(lse[0, t] - math.log(Z)) < 1e-13
        for d in range(D):
            assert abs(out[t, 0, d] - sum(w[j] * v[j, 0, d] for j in range(t + 1)) / Z) < 1e-13


def test_masked_attention_no_visible_key():
    q = np.ones((2, 1, 4), np.float32)
    k = np.ones((3, 1, 4), np.float32)
    out, lse = oracle.attention(q, [0, 5], k, k, [1, 2, 3], 1.0)
    assert lse[0, 0] == -np.inf and np.all(out[0] == 0.0)
    assert np.isfinite(lse[0, 1])


# ---- LSE merge ---------------------------------------------------------------------------

def _split_attention(q, k, v, scale, parts):
    N = q.shape[0]
    outs, lses = [], []
    for idx in parts:
        o, l = oracle.attention(q, np.arange(N), k[idx], v[idx], np.asarray(idx), scale)
        outs.append(o)
        lses.append(l)
    return outs, lses


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_merge_of_disjoint_key_sets_equals_full_attention(nparts):
    """Ring invariant: attention over a union of disjoint key sets equals the
    LSE merge of the attentions over each set.  Pins merge against the attention oracle."""
    N, Hq, Hkv, D = 40, 4, 2, 8
    q, k, v = (t.numpy() for t in qkv(N, Hq, Hkv, D, torch.float32, seed=10))
    rng = np.random.default_rng(0)
    owner = rng.integers(0, nparts, N)
    parts = [np.nonzero(owner == i)[0] for i in range(nparts)]
    outs, lses = _split_attention(q, k, v, 0.4, parts)
    mo, ml = oracle.lse_merge(outs, lses)
    fo, fl = oracle.causal_rows(q, k, v, 0.4)
    np.testing.assert_allclose(mo, fo, atol=1e-13, rtol=0)
    np.testing.assert_allclose(ml, fl, atol=1e-13, rtol=0)


def test_merge_algebra():
    rng = np.random.default_rng(1)
    T, H, D = 16, 3, 8
    os_ = [rng.standard_normal((T, H, D)) for _ in range(3)]
    ls_ = [rng.standard_normal((H, T)) * 5 for _ in range(3)]
    ls_[1][0, :4] = -np.inf
    a = oracle.lse_merge(os_, ls_)
    b = oracle.lse_merge(os_[::-1], ls_[::-1])                     # commutative
    ab = oracle.lse_merge(os_[:2], ls_[:2])
    c = oracle.lse_merge([ab[0], os_[2]], [ab[1], ls_[2]])          # associative
    for x, y in ((a, b), (a, c)):
        np.testing.assert_allclose(x[0], y[0], atol=1e-13)
        np.testing.assert_allclose(x[1], y[1], atol=1e-13)
    # (-inf, anything) is an exact identity
    neg = np.full((H, T), -np.inf)
    e = oracle.lse_merge([os_[0], rng.standard_normal((T, H, D))], [ls_[0], neg])
    np.testing.assert_array_equal(e[0], os_[0])
    np.testing.assert_array_equal(e[1], ls_[0])
    # all -inf: O = 0, lse = -inf, no NaN
    z = oracle.lse_merge([os_[0], os_[1]], [neg, neg])
    assert np.all(z[0] == 0.0) and np.all(z[1] == -np.inf)


# ---- zigzag partition --------------------------------------------------------------

def _golden_zigzag():
    rows = []
    with open(os.path.join(GOLDEN, "zigzag_p75.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append(tuple(int(x) for x in line.split()))
    return rows


def test_zigzag_matches_paper_example():
    for N, inst, a, b in _golden_zigzag():
        m = 3
        tr, ts = oracle.zigzag_map(2 * N * m, N)
        for shard, slot0 in ((a, 0), (b, m)):
            toks = np.arange(shard * m, (shard + 1) * m)
            assert np.all(tr[toks] == inst)
            np.testing.assert_array_equal(ts[toks], slot0 + np.arange(m))


@pytest.mark.parametrize("s", [1, 2, 4, 8])
@pytest.mark.parametrize("m", [1, 3, 8])
def test_zigzag_permutation_and_equal_work(s, m):
    L = 2 * s * m
    tr, ts = oracle.zigzag_map(L, s)
    # permutation: every (rank, slot) used exactly once, 2m tokens per rank
    pairs = set(zip(tr.tolist(), ts.tolist()))
    assert len(pairs) == L
    assert all(0 <= r < s and 0 <= sl < 2 * m for r, sl in pairs)
    # "identical computation workload": causal pairs per rank = m^2 (2s-1) + m (m+1)
    work = np.zeros(s, np.int64)
    np.add.at(work, tr, np.arange(L) + 1)
    assert np.all(work == m * m * (2 * s - 1) + m * (m + 1))
    # contiguous shards (Fig. 1-(b)) are the negative control: imbalanced for s > 1
    cont = np.zeros(s, np.int64)
    np.add.at(cont, np.arange(L) // (2 * m), np.arange(L) + 1)
    if s > 1:
        assert cont.max() > cont.min()


@pytest.mark.parametrize("s", [2, 4, 8])
def test_zigzag_per_step_rule(s):
    """Ring step k: rank r attends to src=(r-k) mod s.  Brute-force visible pairs: step 0
    = 2m^2+m (causal), src<r: all Q x first half of src, src>r: second half of Q x all."""
    m = 4
    pos = oracle.rank_positions(2 * s * m, s)
    for r in range(s):
        for kstep in range(s):
            src = (r - kstep) % s
            vis = pos[src][None, :] <= pos[r][:, None]
            if kstep == 0:
                assert vis.sum() == 2 * m * m + m
            else:
                assert vis.sum() == 2 * m * m
                if src < r:
                    assert vis[:, :m].all() and not vis[:, m:].any()
                else:
                    assert vis[m:, :].all() and not vis[:m, :].any()


def test_zigzag_rejects_ragged():
    with pytest.raises(oracle.OracleError):
        oracle.zigzag_map(10, 4)


# ---- striped partition ---------------------------------

def test_striped_matches_paper_definition_golden():
    """golden/striped_p75.txt: round-robin owners of one-token stripes."""
    n_rows = 0
    with open(os.path.join(GOLDEN, "striped_p75.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            head, owners = line.split("|")
            N, L = (int(x) for x in head.split())
            owners = [int(x) for x in owners.split()]
            tr, ts = oracle.striped_map(L, N)
            assert tr.tolist() == owners
            # within an instance, its tokens keep their order (slot = stripe index)
            for inst in range(N):
                np.testing.assert_array_equal(ts[tr == inst], np.arange(L // N))
            n_rows += 1
    assert n_rows == 4


@pytest.mark.parametrize("s", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [2, 6, 16])
def test_striped_permutation_and_work_closed_form(s, n):
    """Permutation; causal work of rank r = s n(n-1)/2 + n(r+1) for n = L/s tokens per rank
    (sum over its tokens i s + r of i s + r + 1): every rank within n(s-1) pairs of every
    other — near balance, not zigzag's exact balance."""
    L = s * n
    if L % (2 * s):
        pytest.skip("R6: L % 2s == 0")
    tr, ts = oracle.striped_map(L, s)
    assert len(set(zip(tr.tolist(), ts.tolist()))) == L
    work = np.zeros(s, np.int64)
    np.add.at(work, tr, np.arange(L) + 1)
    for r in range(s):
        assert work[r] == s * n * (n - 1) // 2 + n * (r + 1)
    assert work.max() - work.min() == n * (s - 1)


@pytest.mark.parametrize("s", [2, 4, 8])
def test_striped_per_step_shifted_causal(s):
    """Ring step with source src: q row i (position i s + r) sees kv row j (j s + src) iff
    j <= i (src <= r) or j < i (src > r) — a shifted causal mask; brute force."""
    n = 6
    pos = oracle.rank_positions(s * n, s, interleave="striped")
    for r in range(s):
        for src in range(s):
            vis = pos[src][None, :] <= pos[r][:, None]
            i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
            expect = (j <= i) if src <= r else (j < i)
            np.testing.assert_array_equal(vis, expect)
            assert vis.sum() == (n * (n + 1) // 2 if src <= r else n * (n - 1) // 2)


def test_striped_rejects_ragged():
    with pytest.raises(oracle.OracleError):
        oracle.striped_map(12, 4)


def test_striped_plan_stores():
    """Striped chunks append their stripes; balancing (R8) and conservation are unchanged."""
    plan = [(64, [0, 1], "striped"), (64, [0, 1, 2, 3]), (128, list(range(8)), "striped"),
            (32, list(range(8)), "striped")]
    C = 0
    for c in range(len(plan)):
        n, pos, _ = oracle.plan_stores(plan, c)
        np.testing.assert_array_equal(np.sort(np.concatenate(pos)), np.arange(C))
        if C > 0:
            assert n.max() - n.min() <= 1
        C += plan[c][0]
    # chunk 0 (striped over [0, 1]): rank r's store before chunk 1's balancing = r, r+2, ...
    n, pos, _ = oracle.plan_stores([(64, [0, 1], "striped"), (32, [0, 1])], 1)
    for r in range(2):
        np.testing.assert_array_equal(pos[r], np.arange(r, 64, 2))


# ---- cache balancing --------------------------------------------------------------

def test_balancing_matches_fig5():
    plan, moves, store_n = [], [], None
    with open(os.path.join(GOLDEN, "fig5_balancing.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            w = line.split()
            if w[0] == "plan":
                plan.append((int(w[1]), [int(x) for x in w[2:]]))
            elif w[0] == "move":
                moves.append(tuple(int(x) for x in w[1:]))
            elif w[0] == "store_n":
                store_n = [int(x) for x in w[1:]]
    n, pos, mv = oracle.plan_stores(plan, 1)
    assert sorted(mv) == sorted(moves)
    assert n.tolist() == store_n
    # the second half of P_i's chunk-0 store is what P_(i+4) now holds
    n0, pos0, _ = oracle.plan_stores(plan + [(16, list(range(8)))], 1)
    full0 = oracle.rank_positions(4096, 4)
    for i in range(4):
        np.testing.assert_array_equal(pos0[i], full0[i][:512])
        np.testing.assert_array_equal(pos0[i + 4], full0[i][512:])


def _random_plan(rng):
    sizes = [1, 2, 4, 8]
    n_chunks = int(rng.integers(1, 5))
    plan, grp = [], []
    s = int(rng.choice([1, 2]))
    pool = list(rng.permutation(16))
    for _ in range(n_chunks):
        s = int(max(s, rng.choice(sizes)))
        while len(grp) < s:
            grp.append(int(pool.pop()))
        L = 2 * s * int(rng.integers(1, 6))
        plan.append((L, list(grp)))
    return plan


def test_balancing_evenness_and_conservation():
    rng = np.random.default_rng(2)
    for _ in range(200):
        plan = _random_plan(rng)
        C = 0
        for c in range(len(plan)):
            n, pos, _ = oracle.plan_stores(plan, c)
            # evenly re-distributed: within one token
            if C > 0:
                assert n.max() - n.min() <= 1 or len(plan[c][1]) == len(plan[c - 1][1])
            allpos = np.sort(np.concatenate(pos)) if pos else np.array([])
            np.testing.assert_array_equal(allpos, np.arange(C))     # every past token once
            C += plan[c][0]


def test_balancing_even_when_s_grows_every_chunk():
    plan = [(64, [3]), (64, [3, 0]), (128, [3, 0, 5, 1]), (96, [3, 0, 5, 1, 2, 4, 6, 7])]
    for c, expect_C in ((1, 64), (2, 128), (3, 256)):
        n, _, _ = oracle.plan_stores(plan, c)
        assert n.sum() == expect_C and n.max() - n.min() <= 1


@pytest.mark.parametrize("plan", [
    [(16, [0, 1]), (16, [0])],              # SP shrinks
    [(16, [0, 1]), (16, [1, 0, 2, 3])],     # earlier group not a prefix
    [(12, [0, 1, 2])],                      # s not a power of two
    [(18, [0, 1, 2, 3])],                   # L % 2s != 0
    [(16, [0, 0])],                         # duplicate instance
    [(16, [0, 1]), (24, [0, 1, 2, 3, 4, 5])],  # ratio 3
])
def test_balancing_rejects_illegal_plans(plan):
    with pytest.raises(oracle.OracleError) as e:
        oracle.plan_stores(plan, len(plan) - 1)
    assert e.value.rc == oracle.ORACLE_ERR_PLAN


# ---- paged KV writer (R15) ----------------------------------------------------------

@pytest.mark.parametrize("tp,B", [(1, 16), (2, 16), (4, 8), (8, 16)])
def test_paged_write_bijection_and_roundtrip(tp, B):
    rng = np.random.default_rng(3)
    n, Hkv, D = 50, 8, 16
    src = rng.integers(0, 2**16, (n, Hkv, D), dtype=np.uint16)
    pos = rng.permutation(200)[:n] + 7
    n_table = (pos.max() // B) + 1
    num_blocks = n_table + 5
    bt = rng.permutation(num_blocks)[:n_table].astype(np.int32)
    sentinel = np.uint16(0xDEAD)
    caches = [np.full((num_blocks, B, Hkv // tp, D), sentinel, np.uint16) for _ in range(tp)]
    oracle.paged_write(src, pos, tp, B, bt, caches)
    # gather back through the same layout rule = input (round trip)
    for i, p in enumerate(pos):
        for h in range(Hkv):
            t = h * tp // Hkv
            np.testing.assert_array_equal(caches[t][bt[p // B], p % B, h - t * (Hkv // tp)], src[i, h])
    # bijection: exactly n * Hkv rows written, everything else untouched
    written = sum(int(np.any(c != sentinel, axis=-1).sum()) for c in caches)
    assert written == n * Hkv


def test_paged_write_rejects_bad_block_table():
    src = np.zeros((1, 1, 4), np.uint16)
    caches = [np.zeros((2, 4, 1, 4), np.uint16)]
    with pytest.raises(oracle.OracleError):
        oracle.paged_write(src, [100], 1, 4, np.array([0, 1], np.int32), caches)
    with pytest.raises(oracle.OracleError):
        oracle.paged_write(src, [0], 1, 4, np.array([5], np.int32), caches)
