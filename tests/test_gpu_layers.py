"""GPU parity of the layer-wise CDSP prefill ("Cache-Balancing
Latency Overlap", Fig. 6-b): per-layer KV stores, layer l+1's cache balancing issued on the
communicator stream right after layer l's ring, overlapping the caller's FC work.  Every
layer's output must equal the oracle for that layer's inputs, and every layer's balanced
store must be bit-exact (R8), whether balancing ran inline (layer 0) or pre-issued."""
import math

import numpy as np
import pytest
import torch

import oracle
from tolerances import assert_out_close
from cdsp_inputs import qkv, sample_rows
from paper_2511_06247_b200 import api
from paper_2511_06247_b200.driver import run_plan_loopback_layers

pytestmark = pytest.mark.gpu

PLANS = [
    [(512, [0, 1]), (512, [0, 1, 2, 3]), (1024, list(range(8)))],
    [(256, [0]), (256, [0, 1]), (512, [0, 1, 2, 3]), (1024, list(range(8)))],
    [(1024, [3, 1]), (1024, [3, 1, 0, 2])],
]


def _fc(state):
    def between(layer, chunk, rank, stream):
        w = state.setdefault(rank, torch.randn(1024, 1024, device="cuda", dtype=torch.bfloat16))
        for _ in range(3):
            w = (w @ w) * 1e-3  # FC-layer stand-in: the window balancing overlaps
        state[rank] = w
    return between


@pytest.mark.parametrize("plan_list", PLANS)
@pytest.mark.parametrize("with_fc", [False, True])
def test_layers_match_oracle_and_stores_bit_exact(plan_list, with_fc):
    n_layers, Hq, Hkv, D = 3, 8, 2, 128
    N = sum(L for L, _ in plan_list)
    data = [qkv(N, Hq, Hkv, D, torch.bfloat16, seed=70 + l) for l in range(n_layers)]
    plan = api.Plan(plan_list)
    world = max(r for _, rs in plan_list for r in rs) + 1
    cap = api.plan_capacity(plan)
    comms = [api.Comm(i, world, 0, cap, Hkv, D, torch.bfloat16, n_layers=n_layers) for i in range(world)]
    api.connect_local(comms)
    res = run_plan_loopback_layers([tuple(t.cuda() for t in d) for d in data], plan, comms,
                                   between=_fc({}) if with_fc else None)
    torch.cuda.synchronize()
    rows = sample_rows(N, 192, seed=5, edges=[0, N - 1, plan_list[0][0] - 1, plan_list[0][0]]).numpy()
    for l, (q, k, v) in enumerate(data):
        o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                          1.0 / math.sqrt(D), rows=rows)
        o = res[l][0].float().cpu().numpy()[rows]
        lse = res[l][1].cpu().numpy()[:, rows]
        assert_out_close(o, o_ref, True, f"layer {l}")
        assert np.abs(lse - l_ref).max() <= 1e-3, f"layer {l}"
    # every layer's store after the last chunk: the oracle's positions and those rows' K/V
    last_L, last_ranks = plan_list[-1]
    ext = plan_list + [(2 * len(last_ranks), last_ranks)]
    n, pos, _ = oracle.plan_stores(ext, len(plan_list))
    for i, inst in enumerate(last_ranks):
        for l, (q, k, v) in enumerate(data):
            st = comms[inst].kvstore(l)
            assert st.n == n[i]
            np.testing.assert_array_equal(st.pos[: st.n].cpu().numpy().astype(np.int64), pos[i])
            assert torch.equal(st.k[: st.n].cpu(), k[torch.as_tensor(pos[i])]), (inst, l)
            assert torch.equal(st.v[: st.n].cpu(), v[torch.as_tensor(pos[i])]), (inst, l)
    for c in comms:
        c.close()


def test_layer_calls_validate():
    plan = api.Plan([(256, [0, 1])])
    comms = [api.Comm(i, 2, 0, 256, 2, 128, torch.bfloat16, n_layers=2) for i in range(2)]
    api.connect_local(comms)
    q = torch.zeros(128, 4, 128, dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros(128, 2, 128, dtype=torch.bfloat16, device="cuda")
    g = api.SpGroup(comms[0], plan, 0)
    with pytest.raises(api.CdspError) as e:  # layer out of range
        api.prefill_chunk(q, kv, kv, comms[0].kvstore(1), g, layer=2)
    assert e.value.status == 1
    with pytest.raises(api.CdspError) as e:  # store view of another layer
        api.prefill_chunk(q, kv, kv, comms[0].kvstore(0), g, layer=1)
    assert e.value.status == 1
    for c in comms:
        c.close()
