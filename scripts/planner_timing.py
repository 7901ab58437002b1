"""f2: native planner (hc_schedule) time per call vs the paper's Table 6, on the
host it runs on; JSON to stdout."""
import ctypes
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07494_b200 import build

build.build()
from paper_2504_07494_b200 import hc

paper_ms = {50: 0.3, 100: 0.5, 200: 1.0, 400: 2.1, 800: 4.8, 1600: 10.8}
cfg = {"rho": 1.29e-7, "total_units": 0.0, "ttft_slo": 1.5, "tbt_slo": 0.2, "fallback": 1, "eps": 1e-6,
       "decay": 0.4, "hybrid": 1, "block_size": 16}
rs = random.Random(7)
res = {}
for n, ms in paper_ms.items():
    reqs = []
    for i in range(n):
        running = True   # a decode iteration over a memory-tight running batch (hybrid decisions)
        reqs.append({"id": i, "running": int(running), "has_token": int(running), "arrival_time": 1000.0 - rs.uniform(0, 5),
                     "last_token_time": 1000.0 - rs.uniform(0, 0.5), "seq_len": rs.randint(16, 2048)})
    c = dict(cfg, total_units=0.6 * sum(2 * -(-(r["seq_len"] + 1) // 16) for r in reqs))   # KV units at B = 16
    # marshal once (the server keeps its request table in this form), time the C call only
    cc = hc.SchedConfig(*[c[k] for k, _ in hc.SchedConfig._fields_])
    arr = (hc.SchedRequest * n)(*[hc.SchedRequest(*[r[k] for k, _ in hc.SchedRequest._fields_]) for r in reqs])
    a, b, g = (ctypes.c_int32 * n)(), (ctypes.c_int32 * n)(), (ctypes.c_double * n)()
    out = hc.SchedResult()
    call = lambda: hc.lib.hc_schedule(ctypes.byref(cc), n, arr, 1000.0, a, b, g, ctypes.byref(out))
    for _ in range(5):
        assert call() == 0
    t0 = time.perf_counter()
    k = 200
    for _ in range(k):
        call()
    t_c = (time.perf_counter() - t0) / k * 1e3
    t0 = time.perf_counter()
    for _ in range(20):
        hc.schedule(c, reqs, 1000.0)
    t_py = (time.perf_counter() - t0) / 20 * 1e3
    res[n] = {"native_ms": t_c, "with_python_marshalling_ms": t_py, "paper_table6_ms": ms,
              "n_scheduled": int(sum(a)), "n_hidden": int(sum(b))}
print(json.dumps({"metric": "planner time per iteration (hc_schedule, native C++)", "host": os.uname().nodename,
                  "cores": len(os.sched_getaffinity(0)), "candidates": res}, indent=1))
