"""Regenerate profiles/r01_summary.md from the committed profile files."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def line(f):
    return json.loads(open(os.path.join(P, f)).read().strip().splitlines()[-1])


def ncu(f):
    d = {}
    for ln in open(os.path.join(P, f)):
        p = ln.rstrip("\n").split("\t")
        if len(p) == 3:
            d[p[1]] = p[2]
    return d


def row(name, d):
    r, c = d["roofline"], d["clocks"]
    kind = "sustained" if "sustained" in r.get("peak_kind", "") else ("burst" if r["unit"] == "TFLOP/s" else "copy BW")
    return (f"| {name} | {d['ms_per_step']:.3f} | {d['step_ms_percentiles']['p50']:.3f} | {d['value']:.0f} | "
            f"{(d.get('cuda_graph') or {}).get('ms_per_step', float('nan')):.3f} | {r['kernel']} | "
            f"{r['achieved']:.0f} {r['unit']} | {r['frac']:.3f} ({kind}) | {d['step_roofline']['frac']:.3f} | "
            f"{c['sm_mhz']:.0f} MHz, {','.join(c['reasons']) or 'none'} |")


c4, c3, c2, h0 = (line(f"r01_bench_{x}.json") for x in ("cfg4", "cfg3", "cfg2", "cfg5_h0"))
sw = json.load(open(os.path.join(P, "r01_cfg5_sweep.json")))
cub = json.load(open(os.path.join(P, "r01_cublas_same_shapes.json")))
l2 = [json.loads(x) for x in open(os.path.join(P, "r01_l2_fabric_bw.jsonl"))]
cb = c4["cpu_baseline"]
txt = f"""# Round 1 profile summary (B200, sm_100a) — end of round

Peaks: MEASURED_PEAKS.json (re-measured this round) — HBM copy 6543 GB/s; bf16 cuBLAS
1658.7 TF/s burst, 1375.6 TF/s sustained. All timings: CUDA events inside `bench.py`'s
timed region unless marked ncu. Files: `r01_bench_*.json` (bench lines), `r01_launches_cfg4.csv`
(ncu launch list), `r01_ncu_*.txt` (`ncu --set full` details pages), `r01_cfg5_sweep.json`
(hidden-fraction sweep + crossover anatomy), `r01_cublas_same_shapes.json` (library
calibration), `r01_l2_fabric_bw.jsonl` (bulk-copy bandwidth), `r01_rho_calibration.json`,
`traffic.json` (per-launch DRAM bytes and tensor-pipe share used by bench.py),
`r01_pytest_gpu.txt` / `r01_smoke.txt` / `r01_sanitizer_summary.txt`.
Regenerate with `python scripts/make_summary.py`.

## Bench lines (final round-1 code: fused step <3,5,2> with q in registers, 4-n-tile raster)

| workload | ms/step | p50 | req-layers/s | CUDA-graph ms | dominant kernel | achieved | frac of measured peak | step T_roof/T | clocks |
|---|---|---|---|---|---|---|---|---|---|
{row('cfg4 OPT-66B, 256 req, 50% hidden', c4)}
{row('cfg3 OPT-30B, 128 req, planner modes', c3)}
{row('cfg2 OPT-13B, 64 req, 50% hidden', c2)}
{row('cfg5 h=0 (KV only)', h0)}

cfg4 e2e (pinned q in, out + lse back, every step): {c4['e2e']['value']:.0f} req-layers/s; the fp64 oracle
on {cb['cores']} host threads: {cb['value']:.2f} req-layers/s (one thread: {json.dumps(cb.get('single_thread'))}).
Box-to-box spread at cfg4 this round: 40.1-42.3 ms for the fused kernel (SM clock
1305-1447 MHz under the power cap). ncu shows 1.42-1.56 GHz under tensor load even when
nvidia-smi reports 1965 MHz for a short run (cfg2).

## Library calibration and bandwidth probes

cuBLAS (`nvjet_tst_256x256_64x4_2x1_2cta`: the same 256x512 CTA-pair tile) on a dense A of
the same M, N, K: {', '.join(f"{c['shape']} {c['tflops']:.0f} TF/s" for c in cub)}. The
fused kernel (gathered A, attend epilogue, and all KV attention in the same kernel) runs
the GEMM at 1290-1350 TF/s at cfg4.
Bulk-copy streaming into 148 SMs: {', '.join(f"{x['buffer_MiB']} MiB buffer {x['TBps']:.1f} TB/s" for x in l2)}.

## ncu --set full (one launch each)

| kernel (workload) | time | SM clock | DRAM read + write | L2 hit | tensor pipe |
|---|---|---|---|---|---|
"""
for f, name in [("r01_ncu_fused_cfg4.txt", "fused_step_kernel<3,5,2,true> (cfg4)"),
                ("r01_ncu_recon_cfg4.txt", "recon_tc2_kernel<2,4> (cfg4, HC_FUSED=0)"),
                ("r01_ncu_attn_cfg5h0.txt", "attn_pipe_kernel<128,8,3> (cfg5 h=0)")]:
    d = ncu(f)
    txt += (f"| {name} | {d.get('Duration', '')} | {d.get('SM Frequency', '')} | {d.get('dram__bytes_read.sum', '')} + "
            f"{d.get('dram__bytes_write.sum', '')} | {d.get('L2 Hit Rate', '')} | "
            f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', '—')} |\n")
txt += """
The fused kernel's DRAM read varies between captures (46-66 GB per cfg4 launch): the
4-n-tile raster's A-panel sharing depends on how closely the four sharing pairs run.
Attention DRAM read = 1.006 x the algorithmic bytes (K and V rows of 337,276 tokens x 36,864 B).

## Hidden-fraction sweep (cfg5, `r01_cfg5_sweep.json`)

| hidden | ms/step | T_roof/T | SM MHz |
|---|---|---|---|
"""
for h, r in sw["runs"].items():
    txt += f"| {h} | {r['ms_per_step']:.3f} | {r['frac']:.3f} | {r['clocks']['sm_mhz']:.0f} |\n"
txt += """
(Previous commit on a cooler box: `runs_r01e` in the same file, 1/32 at 3.60 ms / 0.57.)
The crossover (1/32) is the weak point: see DESIGN.md §7 "Crossover anatomy".

## f4 (ii) absorbed hidden attention (NON-PAPER variant, `bench.py --absorb`)

cfg4 2.36-2.45 ms/step (104-108 K req-layers/s); `r01_bench_cfg4_absorb.json`, `r01_ncu_absorb_cfg4.txt`,
`r01_cfg5_sweep_absorb.json`.

## NEXT rows f1-f4

| row | file | result |
|---|---|---|
| f1 decode layer (LN off) | `r01_bench_layer_cfg4.json` | cfg4 40.2-41.6 ms/step, 6156-6370 req-layers/s |
| f2 planner (native `hc_schedule`) | `r01_planner_timing.json` | 50: 4 us ... 1600: 196 us (paper Table 6: 0.3 ... 10.8 ms) |
| f3 prefill (OPT-66B, 8 x 2048) | `r01_bench_prefill_8x2048.json`, `r01_ncu_prefill_attn_tc.txt` | 8.9-9.9 ms, 1.66-1.83 M tokens/s |
| f4 (i) RoPE, cfg4 | `r01_bench_cfg4_rope.json` | 41.4-42.6 ms/step |
"""
open(os.path.join(P, "r01_summary.md"), "w").write(txt)
print("wrote profiles/r01_summary.md")
