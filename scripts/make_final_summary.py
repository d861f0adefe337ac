"""Write profiles/r01_final_summary.md from the committed final bench line, the ncu capture of the
default step and the launch list (tooling; run after copying a new measurement set into profiles/)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout


c2 = json.load(open(os.path.join(P, "r01_final_bench_c2.json")))
r = c2["roofline"]
k = r["kernel_ms_per_step"]
out = [f"""# Round 1 — final profiles of the default step (tile-major fast pass, exact-replay escalation)

Captured on one B200 under gpurun, `ncu --set full --clock-control none --import-source on`, command
`python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-mlp` (C2: 200 k posed
points × 24 inits, 32³ grid, max_iters 50), after the same command exited 0 without ncu
(`scripts/gpu_ncu_default.sh`). Per-launch times under ncu are cold-cache and serialised: compare shares,
not absolutes. Report: `r01_final_search.ncu-rep` (k_search_fast, k_esc_start, k_search_escalated<exact>,
k_dedup); launch list `r01_final_launches.csv` (the bench's live FFMA / L1-gather peak probes and the
dense-output scatter are in the list too; the step's kernels are the k_search_* / k_esc_* / k_dedup /
k_sort_* / k_scan_* / k_emit / k_precompute rows). Earlier captures of this round are in git history under
the same names; `r01_search_kernels.ncu-rep`, `r01_ksearch_v1.ncu-rep` and `r01_summary.md` are the first
before/after.

## Bench line this capture explains (`r01_final_bench_c2.json`, timed without ncu)

C2 step {c2['ms_per_step']:.4f} ms = {c2['value']:.3e} solves/s (CUDA graph, L2 flushed between steps, SM clock
{c2['clocks']['sm_mhz']} MHz, no throttle reasons). `k_search_fast` {k['k_search_fast']:.3f} ms: {r['achieved']:.1f} TFLOP/s of
algorithmic FP32 work = {100 * r['frac']:.1f} % of the live-measured FFMA peak ({r['peak']:.1f} TFLOP/s); gather
{r['gather']['achieved_GBps'] / 1e3:.1f} TB/s = {100 * r['gather']['frac']:.0f} % of the measured L1 gather rate. Escalation
`k_esc_start` {k['k_esc_start']:.3f} + `k_search_escalated` {k['k_search_escalated']:.3f} ms for {100 * r['fp64_escalation']['frac_of_solves']:.2f} % of
the solves. e2e through `fsk_deform_host_frames` (host buffers, copies inside): {c2['e2e']['value']:.3e} solves/s;
CPU oracle (f64, {c2['cpu_baseline']['cores']} host threads): {c2['cpu_baseline']['value']:.3e} solves/s.

## What changed during the round's last part (each output bitwise-identical, except the rule change)

* `k_search_fast` 0.633 → 0.549 ms live: tile-major blocks (one CTA solves 8 bone inits of the same 128
  sorted queries back to back): L1 hit 63.6 % → 77.9 %, issue busy 46.5 % → 51.9 %, long-scoreboard
  stalls 38 % → 30 %; J~/meta stored with streaming hints, x/residual with L2 evict-last (DRAM writes
  205 → 180 MB per launch); work counters flushed once per thread instead of 4 atomics per warp per solve.
* `k_esc_start` 0.107 → 0.093 ms (at 4.25 % escalated): one pass over the weight grid (∇w parked in shared memory), 2 CTAs/SM.
* `k_search_escalated<exact>` 0.302 → 0.259 ms (at 4.25 % escalated): 254 registers at 2 CTAs/SM instead of 168 with
  loop-carried spills (the hottest instruction of the old capture was a local-memory reload at the loop
  head).
* Escalation rules: unconverged runs escalate from 5 iterations (was 3), and solves converging on the
  float32 cap iteration with a long last step escalate too — 4.85 % → 5.15 % of the solves; 450-scene
  band study: max |dx| 8.7e-5, 25 mask flips in 324 M solves (`r01_esc_rule_study/`).

## Search kernels

"""]
out.append(run("scripts/ncu_summary.py", os.path.join(P, "r01_final_search.ncu-rep")))
for kname in ("k_search_fast", "k_esc_start", "k_search_escalated"):
    csv = subprocess.run(["ncu", "-i", os.path.join(P, "r01_final_search.ncu-rep"), "--page", "source", "--csv",
                          "--print-source", "sass", "-k", "regex:" + kname], capture_output=True, text=True).stdout
    tmp = f"/tmp/_src_{kname}.csv"
    open(tmp, "w").write(csv)
    out.append(f"\n### {kname} stalls\n```\n" + "\n".join(run("scripts/ncu_stalls.py", tmp).splitlines()[:12]) + "\n```\n")
old = open(os.path.join(P, "r01_final_summary.md")).read()
if "## MLP stages" in old:
    mlp = old[old.index("## MLP stages"):]
    mlp = mlp[:mlp.index("## Launch list")] if "## Launch list" in mlp else mlp
    out.append("\n" + mlp)
out.append("## Launch list of the bench process (`r01_final_launches.csv`, ncu --metrics gpu__time_duration.sum, "
           "incl. the peak probes)\n\n")
out.append(run("scripts/ncu_summary.py", os.path.join(P, "r01_final_launches.csv"), "--launches"))
open(os.path.join(P, "r01_final_summary.md"), "w").write("".join(out))
print("wrote profiles/r01_final_summary.md")
