"""Debug helper: per-request error of the absorbed path vs the oracle on a small case."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_07494_b200 import build
build.build()
from paper_2504_07494_b200 import hc
from tests import hc_testlib as T
from tests.test_gpu_parity import _bf16_workload
from oracle import hc_oracle as O

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,2,128,16").split(","))
n = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 15, 16, 17, 129, 300, 513, 1000, 33, 2]
w = _bf16_workload(*shape, n=n, bias=True)
pool = T.make_pool(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
T.fill(pool, w)
q = T.queries(w)
out, lse = T.decode(pool, w, q)
pool2 = T.make_pool(w)
T.fill(pool2, w)
out2, lse2 = T.decode(pool2, w, q)
H, dh = w.shape.H, w.shape.dh
for i in range(len(w.n)):
    ref, lref = T.oracle_request(w, i)
    e = O.max_rel_err(out[i][None], ref[None], H)
    e2 = O.max_rel_err(out2[i][None], ref[None], H)
    print(i, "mode", w.modes[i], "n", w.n[i], "err absorbed %.3e recon %.3e" % (e, e2),
          "lse", np.abs(lse[i] - lref).max(), "first vals", out[i][:4], ref[:4])
