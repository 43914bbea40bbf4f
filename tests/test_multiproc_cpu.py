"""N>1 host logic on CPU with gloo, world_size 2: IPC-handle exchange, plan-consistency check,
max-over-ranks timing, and that every rank derives the same ring schedule from the plan."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_06247_b200 import api, dist_utils
        res = {}
        blobs = dist_utils.exchange_bytes(bytes([rank]) * 64)
        res["handles"] = [b[0] for b in blobs] == list(range(world)) and all(len(b) == 64 for b in blobs)
        plan = [(4096, [0, 1]), (4096, [0, 1])]
        dist_utils.check_plan_consistent(plan)
        res["plan_ok"] = True
        bad = [(4096, [0, 1])] if rank == 0 else [(8192, [0, 1])]
        try:
            dist_utils.check_plan_consistent(bad)
            res["mismatch_detected"] = False
        except RuntimeError:
            res["mismatch_detected"] = True
        res["max"] = dist_utils.max_over_ranks([float(rank), 10.0 - rank])
        # every rank derives the same partition / balancing schedule (no metadata on the wire)
        P = api.Plan([(2048, [0]), (2048, [0, 1])])
        tr, ts, rp, moves = api.plan_partition(P, 1)
        res["sched"] = (int(tr.sum()), int(ts.sum()), int(rp.sum()), tuple(moves))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_plumbing():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, res = q.get(timeout=120)
        results[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert results[r]["handles"]
        assert results[r]["plan_ok"]
        assert results[r]["mismatch_detected"]
        assert results[r]["max"] == [1.0, 10.0]
    assert results[0]["sched"] == results[1]["sched"]
