"""Diagnostic: max-abs error vs the oracle of a loopback plan under each ring option, with the
location of the worst element and |o_ref| there (rounding-limited or structural?)."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from cdsp_inputs import qkv  # noqa: E402
from paper_2511_06247_b200 import api  # noqa: E402
from paper_2511_06247_b200.driver import make_loopback_comms, run_plan_loopback  # noqa: E402

CASES = {
    "striped_sharp": ([(2048, [0, 1], "striped"), (2048, [0, 1, 2, 3], "striped")], 4096, 4, 2, 128, True, 9),
    "zigzag_sharp": ([(2048, [0, 1]), (2048, [0, 1, 2, 3])], 4096, 4, 2, 128, True, 9),
    "single_sharp": ([(4096, [0])], 4096, 4, 2, 128, True, 9),
}
res = {}
for name, (pl, N, Hq, Hkv, D, sharp, seed) in CASES.items():
    q, k, v = qkv(N, Hq, Hkv, D, torch.bfloat16, seed=seed, sharp=sharp)
    o_ref, l_ref = oracle.causal_rows(q.float().numpy(), k.float().numpy(), v.float().numpy(), 1.0 / math.sqrt(D))
    plan = api.Plan(pl)
    for opt in (0, api.RING_STEPWISE):
        comms = make_loopback_comms(plan, Hkv, D, torch.bfloat16, Hq=Hq)
        for c in comms:
            c.set_ring_options(opt)
        out, lse = run_plan_loopback(q.cuda(), k.cuda(), v.cuda(), plan, comms=comms)
        torch.cuda.synchronize()
        o = out.float().cpu().numpy()
        err = np.abs(o - o_ref)
        i = np.unravel_index(np.argmax(err), err.shape)
        # the error budget at that element: bf16 half-ulp of the output
        ref = o_ref[i]
        half_ulp = 2.0 ** (math.floor(math.log2(abs(ref))) - 8) if ref != 0 else 0
        res[f"{name}_opt{opt}"] = {"max_abs": float(err.max()), "at": [int(x) for x in i], "o_ref": float(ref),
                                   "half_ulp_out": half_ulp, "mean_abs": float(err.mean()),
                                   "p99": float(np.quantile(err, 0.99)),
                                   "lse_max": float(np.abs(lse.cpu().numpy() - l_ref).max())}
        for c in comms:
            c.close()
print(json.dumps(res, indent=1))
