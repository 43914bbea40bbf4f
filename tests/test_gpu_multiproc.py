"""The real multi-process path on one B200: two processes (one instance each) share GPU 0,
exchange cudaIpcMemHandles over a gloo process group, and run an SP=2 plan through
cdsp_prefill_chunk — IPC-mapped stores, device-side peer barriers and copy-engine ring
pulls, exactly as on an 8-GPU box (only the peer pointers are on the same device)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

PLAN = [(1024, [0, 1]), (1024, [0, 1]), (2048, [0, 1])]
N, HQ, HKV, D = 4096, 4, 2, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, plan_list=PLAN, n_layers=None, seed=31):
    """n_layers None: single-store API (cdsp_prefill_chunk); else the layered API, layers called
    in order per chunk with a matmul between them (the FC stand-in the balancing overlaps)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_DEVICE_MAX_CONNECTIONS="32")
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from cdsp_inputs import qkv
        from paper_2511_06247_b200 import api, dist_utils
        dist_utils.check_plan_consistent(plan_list)
        plan = api.Plan(plan_list)
        layers = [None] if n_layers is None else list(range(n_layers))
        comm = api.Comm(rank, world, 0, api.plan_capacity(plan), HKV, D, torch.bfloat16, n_layers=len(layers))
        comm.connect_process_group()
        data = [tuple(t.cuda() for t in qkv(N, HQ, HKV, D, torch.bfloat16, seed=seed + (l or 0))) for l in layers]
        fc = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
        outs = []
        for c, (L, ranks) in enumerate(plan_list):
            if rank not in ranks:
                continue
            C = plan.chunk_start(c)
            s = len(ranks)
            r = ranks.index(rank)
            _, _, rank_pos, _ = api.plan_partition(plan, c)
            for li, l in enumerate(layers):
                qf, kf, vf = data[li]
                qs = api.zigzag_gather(qf[C:C + L].contiguous(), s, r)
                ks = api.zigzag_gather(kf[C:C + L].contiguous(), s, r)
                vs = api.zigzag_gather(vf[C:C + L].contiguous(), s, r)
                o = torch.empty_like(qs)
                lse = torch.empty((HQ, qs.shape[0]), dtype=torch.float32, device="cuda")
                api.prefill_chunk(qs, ks, vs, comm.kvstore(l or 0), api.SpGroup(comm, plan, c), 0.0, o, lse,
                                  layer=l)
                for _ in range(4):
                    fc = fc @ fc * 1e-3  # FC-layer stand-in on the same stream
                outs.append((li, rank_pos[r], o, lse))
            torch.cuda.synchronize()
            comm.check()
        outs = [(li, pos, o.float().cpu().numpy(), lse.cpu().numpy()) for li, pos, o, lse in outs]
        dist.barrier()
        comm.close()
        q.put((rank, outs, None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _run_two(plan_list, n_layers, seed):
    import oracle
    from tolerances import assert_out_close
    from cdsp_inputs import qkv
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, plan_list, n_layers, seed)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, outs, err = q.get(timeout=300)
        assert err is None, f"rank {r}: {err}"
        res[r] = outs
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = [qkv(N, HQ, HKV, D, torch.bfloat16, seed=seed + li) for li in range(n_layers or 1)]
    checked = 0
    for r in range(world):
        for li, pos, o, lse in res[r]:
            qf, kf, vf = data[li]
            sel = pos[:: max(1, len(pos) // 96)]
            o_ref, l_ref = oracle.causal_rows(qf.float().numpy(), kf.float().numpy(), vf.float().numpy(),
                                              1.0 / math.sqrt(D), rows=sel)
            idx = np.searchsorted(pos, sel) if np.all(np.diff(pos) > 0) else np.array([list(pos).index(x) for x in sel])
            assert_out_close(o[idx], o_ref, True, f"rank {r} layer {li}")
            assert np.abs(lse[:, idx] - l_ref).max() <= 1e-3, (r, li)
            checked += 1
    assert checked == sum(len(ranks) for _, ranks in plan_list) * (n_layers or 1)


def test_two_processes_ipc_ring_matches_oracle():
    _run_two(PLAN, None, 31)


def test_two_processes_layered_balancing_acks():
    """Layered API across processes with a growing group (s 1 -> 2): layer 0 balances inline,
    layers 1, 2 are pre-balanced on the comm stream during the previous layer, and the old
    rank overwrites the moved half only after the new rank's cross-process acknowledgement."""
    _run_two([(1024, [0]), (1024, [0, 1]), (2048, [0, 1])], 3, 41)


def test_bench_torchrun_two_ranks_one_gpu():
    """bench.py's N>1 path (torchrun, IPC ring, max-over-ranks timing) runs end to end and
    prints one JSON line from rank 0 (both ranks pinned to GPU 0: functional check only)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CDSP_BENCH_DEVICE="0", CUDA_DEVICE_MAX_CONNECTIONS="32")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--seq", "4096", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["sp"] == 2 and d["value"] > 0
    ring = d["ring"]
    for key in ("pull_gbs", "exposed_ms_per_step", "control_ms_per_step", "hidden_ms", "bytes_per_step"):
        assert ring[key] is not None, key
    assert ring["control_ms_per_step"] > 0 and ring["pull_gbs"] > 0
    assert d["roofline"]["launches_timed"] == 2  # one fused ring launch per step
    assert d["gpu_launches"] == 2 * 9


def test_bench_torchrun_eight_ranks_one_gpu():
    """bench.py at N = 8 (the SCALE run's largest size): eight processes, an SP = 8 ring of
    CUDA-IPC stores, device peer barriers and copy-engine pulls, max-over-ranks timing — all
    pinned to GPU 0 (functional check only: the ranks time-slice one GPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CDSP_BENCH_DEVICE="0", CUDA_DEVICE_MAX_CONNECTIONS="32")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "8",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "8", "--steps", "2", "--warmup", "1", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 8 and d["config"]["sp"] == 8 and d["value"] > 0
    assert d["ring"]["pulls_per_step"] == 7 and d["ring"]["pull_gbs"] > 0
    assert d["roofline"]["launches_timed"] == 2 and d["roofline"]["traffic"] is not None


def test_bench_weak_is_configs4_shape():
    """--weak: GQA 32/8 with 64K tokens per GPU (at N = 8 this is configs[4]'s 512K prompt)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CDSP_BENCH_DEVICE="0", CUDA_DEVICE_MAX_CONNECTIONS="32")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--weak", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    c = d["config"]
    assert (c["prompt_tokens"], c["q_heads"], c["kv_heads"], c["sp"]) == (131072, 32, 8, 2)
    assert d["scaling"] == "weak" and d["ring"]["hidden_ms"] is not None


def _geometry_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2511_06247_b200 import api
        comm = api.Comm(rank, world, 0, 1024, 2, 128, torch.bfloat16, n_layers=1 + rank)  # layers differ
        try:
            comm.connect_process_group()
            q.put((rank, "connected"))
        except api.CdspError as e:
            q.put((rank, e.status))
        dist.barrier()
        comm.close()
    finally:
        dist.destroy_process_group()


def test_connect_refuses_mismatched_geometry():
    """A peer created with another n_layers is refused (CDSP_ERR_COMM) instead of mapping its
    store at offsets computed from this instance's geometry."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_geometry_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: 7, 1: 7}
