"""Write profiles/r02_final_summary.md from the round-2 measurement set (tooling; run after copying
the set into profiles/: r02_final_bench_*.json, r02_final_search.ncu-rep, r02_final_launches.csv)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout


def load(tag):
    return json.load(open(os.path.join(P, f"r02_final_bench_{tag}.json")))


c2, c3, c3d, c4, c5, ref = (load(t) for t in ("c2", "c3", "c3det", "c4", "c5", "ref"))
r = c2["roofline"]
k = r["kernel_ms_per_step"]
esc = r["fp64_escalation"]
k3 = c3["roofline_k3"]
e = c2["e2e"]


def row(name, d, note=""):
    ee = d.get("e2e") or {}
    e2e = f"{ee['value']:.3e}" if ee.get("value") else "—"
    return f"| {name} | {d['ms_per_step']:.4f} | {d['value']:.3e} | {e2e} | {note} |\n"


out = [f"""# Round 2 — final measurement set and profiles

One B200 under gpurun (SM clock {c2['clocks']['sm_mhz']:.0f} MHz, no throttle reasons on any line). Bench lines are
timed without a profiler (CUDA graph, L2 flushed between steps); ncu numbers come from separate runs of the same
commands after those exited 0 (`scripts/gpu_r2_final.sh`): `r02_final_search.ncu-rep` (`--set full
--clock-control none --import-source on`, one C3 step: k_precompute_v, k_search_fast, k_esc_start,
k_search_escalated<exact>, k_dedup, k_bwd_scatter_agg) and the launch list `r02_final_launches.csv`
(`--metrics gpu__time_duration.sum`, two C2 steps plus the bench's peak probes). ncu per-launch times are
cold-cache and serialised: compare shares, not absolutes.

## Bench lines (`r02_final_bench_*.json`)

| workload | ms / step | solves/s | e2e solves/s (host buffers, copies inside) | note |
|---|---|---|---|---|
"""]
out.append(row("C2: 200 k × 24, 32³ (bench default)", c2, f"{100 * esc['frac_of_solves']:.2f} % of solves re-solved in float64"))
out.append(row("C3: C2 + implicit-diff backward", c3))
out.append(row("C3, deterministic backward", c3d))
out.append(row("C4: 16 poses × 1 M points, 64³ (fsk_deform_frames)", c4))
out.append(row("C5 per-GPU shard: 8 M ray samples (64 per ray), 128×128×32", c5))
out.append(row("reference arm (`--impl reference`, reference sources on all host threads)", ref,
               f"{ref['cpu_baseline']['cores']} threads, {ref['cpu_baseline'].get('kind')}"))
out.append(f"""
C2 e2e (`fsk_deform_host_frames`, {e['frames_per_call']} frames per call, {e['h2d_bytes_per_step'] / 1e6:.1f} MB H2D +
{e['d2h_bytes_per_step'] / 1e6:.1f} MB D2H per frame inside the timing): {e['value']:.3e} solves/s =
{e['value'] / ref['value']:.0f}× the reference arm. One synchronous `fsk_deform_host` call per frame:
{e['single_frame_call']['value']:.3e}. Through the reference-facing C++ API (`fskin::batch_search`, host f64 queries in,
`std::vector<CorrespondenceSet>` out): {e['cpp_api']['value']:.3e} solves/s.

## Rooflines

* `k_search_fast` (K2, float32 pass): {k['k_search_fast']:.4f} ms, {r['achieved']:.1f} TFLOP/s algorithmic =
  {100 * r['frac']:.1f} % of the live FFMA peak ({r['peak']:.1f}); gathers {r['gather']['achieved_GBps'] / 1e3:.1f} TB/s =
  {100 * r['gather']['frac']:.0f} % of the measured L1 gather rate; DRAM traffic {r['traffic'] / 1e6:.0f} MB per launch.
* Escalation: `k_esc_start` {k['k_esc_start']:.4f} + `k_search_escalated` {k['k_search_escalated']:.4f} ms for
  {esc['solves']:.0f} solves ({esc['iterations']:.0f} float64 iterations, {esc['achieved_TFLOPs_f64']:.2f} TFLOP/s f64 of
  {esc['peak_TFLOPs_f64_measured']:.1f} measured).
* `k_bwd_scatter_agg` (K3, C3): {1e3 * k3['avg_launch_ms']:.1f} µs, {k3['achieved']:.0f} GB/s of algorithmic reductions
  = {100 * k3['frac']:.0f} % of the measured RED.F32x4 rate ({k3['peak']:.0f} GB/s).
* K1 `k_precompute_v` (C5 grid, the one large enough to stream): see `r02_final_bench_c5.json` `roofline.k1`
  ({100 * c5['roofline']['k1']['frac_of_hbm_moved']:.0f} % of HBM on the bytes it moves).

## Search kernels (ncu)

""")
out.append(run("scripts/ncu_summary.py", os.path.join(P, "r02_final_search.ncu-rep")))
for kname in ("k_search_fast", "k_esc_start", "k_search_escalated", "k_bwd_scatter_agg"):
    csv = subprocess.run(["ncu", "-i", os.path.join(P, "r02_final_search.ncu-rep"), "--page", "source", "--csv",
                          "--print-source", "sass", "-k", "regex:" + kname], capture_output=True, text=True).stdout
    tmp = f"/tmp/_src_{kname}.csv"
    open(tmp, "w").write(csv)
    out.append(f"\n### {kname} stalls\n```\n" + "\n".join(run("scripts/ncu_stalls.py", tmp).splitlines()[:12]) + "\n```\n")
out.append("""
## What the round changed (measured; details and the rejected ones in DESIGN.md §4a″)

Kept: FFMA2 trilinear accumulate (K2 0.549 → 0.542 ms); K1 one thread per vertex with whole x-pair row
stores (C5 K1 101 → 70 µs, 49 % of HBM); host pipeline on cached CUDA graphs and staged (sort + K1 of
item i+1 beside item i's search): C2 e2e 4.67e9 → 4.93e9; `fsk_deform_frames` (C4 68.2 → 67.9 ms);
look-back scan; K3 records in shared memory; deterministic backward one product per record and lane
(49.7 → 29.0 µs); 512-thread MLP CTAs (MLP-variant search 28.1 → 23.1 ms); escalation rules found by
full-workload and 1 950-scene band studies: conditioning max|J~| > 5, stagnation + max|J~| > 2.5, init on a
cell face (a 0.22-off root), transient J~ spike > 7 (roots 1.1–1.9e-4 off; costs +1 % C2 step in register
spill) — after them no converged root beyond 8.9e-5 in 1.40 G band-study solves, and the full C4/C5
workloads within 9.8e-5 of the reference's own code.

Measured and rejected (bitwise-equal outputs, slower): next-init L1 prefetch (+7 %), fused cooperative
sort, cp.async-prefetched refill, TMA bulk dedup, L2 set-aside, ordered deterministic backward, smaller
host chunks, float32 cap 9–12 (faster, but the band study finds roots up to 4.1e-4 off), exact-replay
corner prefetch, FMUL2 weight pairs, single-block sort scan; shared-memory staging of the tile sub-grid
was studied (`r02_staging_study.log`) and not built.
""")
out.append("\n## Launch list (`r02_final_launches.csv`, incl. the peak probes)\n\n")
out.append(run("scripts/ncu_summary.py", os.path.join(P, "r02_final_launches.csv"), "--launches"))
open(os.path.join(P, "r02_final_summary.md"), "w").write("".join(out))
print("wrote profiles/r02_final_summary.md")
