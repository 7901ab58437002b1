"""Copy a profile_round.sh output directory (gpurun_out/<tag>) into profiles/: the cfg4 bench
line and launch list, text summaries of the ncu --set full captures, and traffic.json
(dram bytes and tensor-pipe share per launch, read by bench.py)."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles")
NCU = "/usr/local/cuda/bin/ncu"
SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy", "Launch Statistics",
            "Scheduler Statistics", "Compute Workload Analysis")


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def details(rep, title, out_name):
    out = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    idx = {h: i for i, h in enumerate(rows[0])}
    lines = [f"{r[idx['Section Name']]}\t{r[idx['Metric Name']]}\t{r[idx['Metric Value']]} {r[idx['Metric Unit']]}"
             for r in rows[1:] if len(r) > idx["Metric Value"] and r[idx["Section Name"]] in SECTIONS]
    m = raw(rep)
    keys = ["dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]
    lines += [f"raw\t{k}\t{m[k][0]} {m[k][1]}" for k in keys if k in m]
    open(os.path.join(dst, out_name), "w").write(title + "\n" + "\n".join(lines) + "\n")
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    nbytes = sum(float(m[k][0]) * scale[m[k][1]] for k in keys[:2])
    return nbytes, float(m[keys[2]][0])


shutil.copy(os.path.join(src, "bench_cfg4.json"), os.path.join(dst, "r01_bench_cfg4.json"))
shutil.copy(os.path.join(src, "bench_cfg5_h0.json"), os.path.join(dst, "r01_bench_cfg5_h0.json"))
shutil.copy(os.path.join(src, "launches_cfg4.csv"), os.path.join(dst, "r01_launches_cfg4.csv"))
fb, ft = details(os.path.join(src, "full_fused_cfg4.ncu-rep"),
                 "# ncu --set full: fused_step_kernel<3,5,2,true> (q in registers), attend epilogue (cfg4: OPT-66B, 256 req, 50% hidden)",
                 "r01_ncu_fused_cfg4.txt")
rb, rt = details(os.path.join(src, "full_recon_cfg4.ncu-rep"),
                 "# ncu --set full: recon_tc2_kernel<2,4>, attend epilogue (HC_FUSED=0, cfg4)", "r01_ncu_recon_cfg4.txt")
ab, _ = details(os.path.join(src, "full_attn_cfg5h0.ncu-rep"),
                "# ncu --set full: attn_pipe_kernel<128,8,3> (cfg5 h=0, KV only)", "r01_ncu_attn_cfg5h0.txt")
json.dump({"_source": f"ncu --set full --clock-control none, one launch each ({tag}; profiles/r01_ncu_*.txt): "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch; *_tensor_pipe_pct: "
                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "cfg4-opt66b": {"fused_step": fb, "fused_step_tensor_pipe_pct": ft, "recon_gemm": rb,
                           "recon_gemm_tensor_pipe_pct": rt},
           "cfg5-opt66b-h0.0000": {"attention": ab}}, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
print("saved", tag, fb, ft, rb, rt, ab)
