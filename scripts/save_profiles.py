"""Copy a profile_round.sh output directory (gpurun_out/<tag>) into profiles/: the bench lines
and launch list, text summaries of the ncu --set full captures, and traffic.json (DRAM bytes
and tensor-pipe share per launch, read by bench.py for the roofline object's `traffic`)."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles")
NCU = "/usr/local/cuda/bin/ncu"
SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Launch Statistics",
            "Scheduler Statistics", "Compute Workload Analysis")
KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "gpu__time_duration.sum"]


def _page(rep, page):
    """ncu page as CSV text: from a .ncu-rep, or from the <name>.<page>.csv export next to it."""
    exp = rep[:-len(".ncu-rep")] + f".{page}.csv"
    if os.path.exists(exp):
        return open(exp).read()
    return subprocess.run([NCU, "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(_page(rep, "raw").splitlines()))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def details(rep, title, out_name):
    out = _page(rep, "details")
    rows = list(csv.reader(out.splitlines()))
    idx = {h: i for i, h in enumerate(rows[0])}
    lines = [f"{r[idx['Section Name']]}\t{r[idx['Metric Name']]}\t{r[idx['Metric Value']]} {r[idx['Metric Unit']]}"
             for r in rows[1:] if len(r) > idx["Metric Value"] and r[idx["Section Name"]] in SECTIONS]
    m = raw(rep)
    lines += [f"raw\t{k}\t{m[k][0]} {m[k][1]}" for k in KEYS if k in m]
    open(os.path.join(dst, out_name), "w").write(title + "\n" + "\n".join(lines) + "\n")
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    nbytes = sum(float(m[k][0]) * scale[m[k][1]] for k in KEYS[:2])
    return nbytes, float(m[KEYS[2]][0]) if KEYS[2] in m else None


for name in os.listdir(src):
    if name.startswith("bench_") and name.endswith(".json") and os.path.getsize(os.path.join(src, name)):
        shutil.copy(os.path.join(src, name), os.path.join(dst, f"{tag}_{name}"))
for name in ("launches_cfg4.csv", "smoke.txt"):
    if os.path.exists(os.path.join(src, name)):
        shutil.copy(os.path.join(src, name), os.path.join(dst, f"{tag}_{name}"))
caps = {
    "full_fused_cfg4": ("# ncu --set full: fused_step_kernel (cfg4: OPT-66B layer, 256 requests, 50% hidden)",
                        "cfg4-opt66b", "fused_step"),
    "full_fused_cfg5_h1_32": ("# ncu --set full: fused_step_kernel at the crossover (cfg5, 1/32 of requests hidden)",
                              "cfg5-opt66b-h0.0312", "fused_step"),
    "full_fused_llama3": ("# ncu --set full: fused_step_kernel, GQA (LLaMA-3-8B layer, 32/8 heads, tensor-core KV loop)",
                          "gqa-llama3-8b", "fused_step"),
    "full_attn_cfg5h0": ("# ncu --set full: attn_pipe_kernel<128,8,3> (cfg5 h=0, KV only)",
                         "cfg5-opt66b-h0.0000", "attention"),
}
traffic = {"_source": f"ncu --set full --clock-control none, one launch each ({tag}; profiles/{tag}_ncu_*.txt): "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch; *_tensor_pipe_pct: "
                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"}
for rep, (title, wl, kern) in caps.items():
    path = os.path.join(src, rep + ".ncu-rep")
    if not os.path.exists(path) and not os.path.exists(os.path.join(src, rep + ".details.csv")):
        print("missing", rep)
        continue
    nb, tp = details(path, title, f"{tag}_ncu_{rep[5:]}.txt")
    traffic.setdefault(wl, {})[kern] = nb
    if tp is not None and kern != "attention":
        traffic[wl][kern + "_tensor_pipe_pct"] = tp
json.dump(traffic, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
