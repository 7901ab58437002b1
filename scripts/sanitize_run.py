"""Small decode runs for compute-sanitizer (tiny fp32, bf16 with every kernel path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import configs as C
from synth.configs import LayerShape, Workload, MODE_KV, MODE_HIDDEN
from tests import hc_testlib as T
from paper_2504_07494_b200 import hc

def run(w, flags=0, split=0):
    pool = T.make_pool(w, flags=flags, split_tokens=split)
    T.fill(pool, w)
    out, lse = T.decode(pool, w, T.queries(w))
    err, _ = T.compare(w, out, lse, range(len(w.n)))
    print(w.name, hex(flags), split, "err", err, flush=True)

run(C.tiny())
run(C.tiny(block_size=4, bias=True))
shape = LayerShape("san", 512, 4, 128)
n = [1, 17, 300, 129, 64, 511, 33]
w = Workload("san-bf16", shape, 16, "bf16", 5, n, [0, 1, 0, 1, 1, 0, 1], list(range(len(n))), True)
run(w)
run(w, split=16)
run(w, flags=hc.HC_FLAG_FORCE_SIMT)
run(w, flags=hc.HC_FLAG_GENERIC_ATTN)
shape64 = LayerShape("san64", 512, 8, 64)
w64 = Workload("san-bf16-dh64", shape64, 32, "bf16", 6, n, [0, 1, 0, 1, 1, 0, 1], list(range(len(n))), False)
run(w64)
torch.cuda.synchronize()
print("done")
