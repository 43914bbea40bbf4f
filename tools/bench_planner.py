"""CDSP scheduler latency (Table 2: avg 22.8-30.6 us, max <= 86.8 us
per call on the authors' host).  Calls cdsp_schedule_prefill on pre-marshalled arguments (only
the ctypes call itself is timed) for random requests and queue states: pools of 8 / 16 / 32
instances (8 per node), SP sizes {1,2,4,8}.  Prints one JSON line.  CPU only."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2511_06247_b200 import api  # noqa: E402


def _case(rng):
    """Seeded request: Eq. (1) coefficients per SP size, a granule-aligned prompt length."""
    models = {}
    for s in (1, 2, 4, 8):
        f = 1.0 / s ** rng.uniform(0.8, 1.0)
        models[s] = (rng.uniform(0.5, 3.0) * (1 + 0.1 * s), rng.uniform(1e-4, 4e-4) * f,
                     rng.uniform(1e-9, 4e-9) * f, rng.uniform(0.5e-9, 2e-9) * f)
    granule = 2 * 8 * int(rng.choice([64, 128]))
    return granule * int(rng.integers(1, 64)), models, float(rng.choice([0.0, 0.05, 0.1, 0.3, 0.5])), granule


def main():
    L_ = api.lib()
    res = {}
    for n_inst in (8, 16, 32):
        rng = np.random.default_rng(n_inst)
        args = []
        while len(args) < 1000:
            L, models, rate, granule = _case(rng)
            q = rng.exponential(100.0, n_inst) * (rng.random(n_inst) < 0.7)
            qa = (ctypes.c_double * n_inst)(*q)
            sizes = sorted(models)
            sz = (ctypes.c_int32 * 4)(*sizes)
            ms = (api.LatencyModel * 4)(*[api.LatencyModel(*models[s]) for s in sizes])
            args.append((L, qa, sz, ms, rate, granule, api.ScheduleC()))
        ts = []
        for L, qa, sz, ms, rate, granule, out in args:
            t0 = time.perf_counter_ns()
            rc = L_.cdsp_schedule_prefill(L, n_inst, ctypes.cast(qa, ctypes.c_void_p), 8, 4,
                                          ctypes.cast(sz, ctypes.c_void_p), ctypes.cast(ms, ctypes.c_void_p),
                                          rate, granule, ctypes.byref(out))
            ts.append((time.perf_counter_ns() - t0) / 1e3)
            assert rc == 0
        ts = np.array(ts[10:])
        res[f"pool{n_inst}"] = {"avg_us": float(ts.mean()), "p50_us": float(np.median(ts)),
                                "p99_us": float(np.quantile(ts, 0.99)), "max_us": float(ts.max())}
    print(json.dumps({"metric": "cdsp_schedule_prefill latency per call (us), host CPU",
                      "cpu": os.uname().machine, "results": res,
                      "paper_table2": "avg 22.8-30.6 us, max 45.1-86.8 us (max SP 8..128)"}))


if __name__ == "__main__":
    main()
