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
# absorbed hidden attention (f4 ii): tcgen05 score / Z kernels, P rescale, q~ / W_V GEMMs
run(w, flags=hc.HC_FLAG_ABSORB_HIDDEN)
run(w64, flags=hc.HC_FLAG_ABSORB_HIDDEN)
# decode layer + prefill (tcgen05 prefill attention) with LayerNorm and RoPE
from oracle import hc_oracle as O
dev = torch.device("cuda", 0)
for ln, rope in ((True, 0.0), (False, 10000.0)):
    wl = Workload("san-layer", shape, 16, "bf16", 7, [1, 40, 130, 300], [0, 1, 0, 1], [0, 1, 2, 3], True)
    pool = T.make_layer_pool(wl, ln=ln, rope_theta=rope)
    x = torch.cat([wl.x(i, device=dev) for i in range(len(wl.n))]).contiguous()
    y = pool.prefill_layer(wl.req_ids, wl.modes, wl.n, x, wl.scale)
    xt = torch.stack([wl.x_t(i, device=dev) for i in range(len(wl.n))]).contiguous()
    y2, _ = pool.decode_layer(wl.req_ids, wl.modes, xt, wl.scale)
    torch.cuda.synchronize()
    print("layer ln", ln, "rope", rope, "finite", bool(torch.isfinite(y).all() and torch.isfinite(y2).all()), flush=True)
# GQA (f4 (i)): fused kernel with the tensor-core KV loop, and the stand-alone tc attention kernel
shg = LayerShape("san-gqa", 1024, 8, 128, 2)
wg = Workload("san-gqa", shg, 16, "bf16", 8, n, [0, 1, 0, 1, 1, 0, 1], list(range(len(n))), True)
run(wg)
run(Workload("san-gqa-kv", shg, 16, "bf16", 9, n, [0] * len(n), list(range(len(n))), False))
# GQA with groups of 8 query heads: rebuilt K/V scratch + the tensor-core loop on hidden tasks
shg8 = LayerShape("san-gqa8", 2048, 16, 128, 2)
run(Workload("san-gqa8", shg8, 16, "bf16", 11, n, [0, 1, 0, 1, 1, 0, 1], list(range(len(n))), True))
# tensor-core KV loop forced on a multi-head pool (knobs are read at pool create)
os.environ["HC_ATTN_TC"] = "2"
run(w)
run(Workload("san-kv", shape, 16, "bf16", 10, n, [0] * len(n), list(range(len(n))), False))
os.environ.pop("HC_ATTN_TC")
torch.cuda.synchronize()
print("done")
