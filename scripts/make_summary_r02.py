"""Regenerate profiles/r02_summary.md from the committed round-2 profile files."""
import json
import os

P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles") + "/"


def L(f):
    return json.loads(open(P + f).read().strip().splitlines()[-1])


def ncu(f):
    d = {}
    for ln in open(P + f):
        p = ln.rstrip("\n").split("\t")
        if len(p) == 3:
            d[p[1]] = p[2]
    return d


rows = [("cfg4 OPT-66B, 256 req, 50% hidden", "r02_bench_cfg4.json"),
        ("cfg3 OPT-30B, 128 req, planner modes", "r02_bench_cfg3.json"),
        ("cfg2 OPT-13B, 64 req, 50% hidden", "r02_bench_cfg2.json"),
        ("LLaMA-3-8B layer (GQA 32/8), 256 req, 50% hidden", "r02_bench_llama3-8b.json"),
        ("LLaMA-3-8B layer + RoPE (theta 5e5)", "r02_bench_llama3-8b_rope.json"),
        ("Yi-6B layer (GQA 32/4), 256 req, 50% hidden", "r02_bench_yi-6b.json"),
        ("cfg4, absorbed variant (NON-PAPER)", "r02_bench_cfg4_absorb.json")]
t = """# Round 2 profile summary (B200, sm_100a) — end of round (final code)

Peaks: MEASURED_PEAKS.json — HBM copy 6533 GB/s; bf16 cuBLAS 1659.5 TF/s burst, 1374.6 TF/s
sustained. Timings: CUDA events inside `bench.py`'s timed region (ncu numbers marked).
Files: `r02_bench_*.json` (bench lines), `r02_launches_cfg4.csv` (ncu launch list),
`r02_ncu_*.txt` (`ncu --set full` details + raw DRAM/tensor-pipe counters), `r02_cfg5_sweep.json`
(hidden-fraction sweep), `r02_*_ab.txt` (same-box A/Bs of this round's changes),
`r02_kv_sm_bw.jsonl` (per-SM bulk-copy bandwidth), `r02_ncu_source_fused_cfg5_h1_32.txt`
(warp-stall samples per code region), `r02_sanitizer_summary.txt`, `r02_pytest_gpu*.txt`, `traffic.json`.
Regenerate with `python scripts/make_summary_r02.py`.

Late-round changes: KV warp loop producer without per-chunk integer divisions and knob
branches (1/64 -1..-5%, 1/32 -1..-4%); dynamic GEMM tile schedule through a cluster tile queue
(cfg4 -1..-2%, 1/32 -2..-6%, 1/16 -4..-5%); GQA attend epilogue on mma.sync (LLaMA-3-8B -6%,
Yi-6B -4%).

## Bench lines

| workload | ms/step | req-layers/s | e2e req-layers/s | dominant kernel (config chosen by the runtime) | achieved | roofline frac | step T_roof/T | clocks |
|---|---|---|---|---|---|---|---|---|
"""
for name, f in rows:
    if not os.path.exists(P + f):
        continue
    d = L(f)
    r, c = d["roofline"], d["clocks"]
    t += (f"| {name} | {d['ms_per_step']:.3f} | {d['value']:.0f} | {d['e2e']['value']:.0f} | {r.get('kernel')} | "
          f"{r['achieved']:.0f} {r['unit']} | {r['frac']:.3f} | {d['step_roofline']['frac']:.3f} | "
          f"{c['sm_mhz']:.0f} MHz, {','.join(c['reasons']) or 'none'} |\n")
t += """
`roofline frac` is against the sustained bf16 peak for power-capped runs and the burst peak
when the SM clock held its maximum or the kernel ran faster than the sustained figure
(`frac_vs_burst` / `frac_vs_sustained` are both in each line).

## ncu (one cold launch each, `--clock-control none`)

| capture | duration | SM clock | tensor pipe | DRAM read | issue slots busy |
|---|---|---|---|---|---|
"""
for name, f in [("fused, cfg4", "r02_ncu_fused_cfg4.txt"), ("fused, cfg5 1/32", "r02_ncu_fused_cfg5_h1_32.txt"),
                ("fused, LLaMA-3-8B", "r02_ncu_fused_llama3.txt"), ("attention, cfg5 h=0", "r02_ncu_attn_cfg5h0.txt")]:
    d = ncu(f)
    t += (f"| {name} | {d.get('Duration', '')} | {d.get('SM Frequency', '')} | "
          f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', '—')} | "
          f"{d.get('dram__bytes_read.sum', '')} | {d.get('Issue Slots Busy', '')} |\n")
sw = json.load(open(P + "r02_cfg5_sweep.json"))
t += ("\n## cfg5 hidden-fraction sweep (T_roof / T per hidden fraction, sustained protocol)\n\n"
      "| hidden | ms/step | T_roof ms | T_roof/T | SM MHz |\n|---|---|---|---|---|\n")
for h, r in sw["points"].items():
    t += f"| {h} | {r['ms_per_step']:.3f} | {r['T_roof_ms']:.3f} | {r['frac']:.3f} | {r['clocks']['sm_mhz']:.0f} |\n"
t += """
The crossover (1/32) is still the weak point (0.58 here vs 0.55 at mid-round on a box that
held similar clocks). DESIGN.md §7 has the measurements behind it: the spatial SM split
(reverted), the KV warp loop's per-chunk cost (ncu warp-stall samples), the per-SM bulk-copy
rates, and the L2 account of the cfg4 DRAM traffic.
"""
open(P + "r02_summary.md", "w").write(t)
print("wrote profiles/r02_summary.md")
