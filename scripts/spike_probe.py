"""Step-time spike probe: the bench.py decode loop (no sync inside the timed region) with
and without the nvidia-smi sampler and the runtime's per-kernel profiling events; prints
the slowest step intervals so host-side stalls (GPU idle between steps) stand out."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_07494_b200 import hc  # noqa: E402
from synth import configs as C  # noqa: E402
from tests import hc_testlib as T  # noqa: E402


def run(pool, w, q, out, lse, ws, steps, smi, prof):
    s = torch.cuda.current_stream()
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL) if smi else None
    time.sleep(0.3)
    pool.set_profiling(prof)
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    host = []
    evs[0].record(s)
    for i in range(steps):
        t0 = time.perf_counter()
        hc.hc_decode_attention(pool.handle, list(w.req_ids), q, w.scale, out, lse, ws, s)
        host.append((time.perf_counter() - t0) * 1e3)
        evs[i + 1].record(s)
    torch.cuda.synchronize()
    pool.set_profiling(False)
    pool.kernel_times()
    if p:
        p.terminate()
        p.wait()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    srt = sorted(per)
    return {"smi": smi, "prof": prof, "mean": sum(per) / steps, "p50": srt[steps // 2], "max": srt[-1],
            "slowest": sorted(range(steps), key=lambda i: -per[i])[:3], "host_max_ms": max(host),
            "host_slowest": sorted(range(steps), key=lambda i: -host[i])[:3]}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    w = C.by_name(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
    pool = T.make_pool(w)
    T.fill(pool, w)
    q = T.queries(w)
    out = torch.empty((len(w.n), w.shape.d), dtype=w.torch_dtype, device="cuda")
    lse = torch.empty((len(w.n), w.shape.H), dtype=torch.float32, device="cuda")
    ws = pool.workspace(list(w.req_ids))
    for _ in range(3):
        hc.hc_decode_attention(pool.handle, list(w.req_ids), q, w.scale, out, lse, ws, torch.cuda.current_stream())
    for rep in range(3):
        for smi, prof in ((True, True), (False, True), (True, False), (False, False)):
            print(json.dumps(run(pool, w, q, out, lse, ws, 50, smi, prof)), flush=True)
