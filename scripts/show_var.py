"""Summarise gpurun_out/var_*.log bench lines (tuning sweeps): step time and per-kernel ms."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/var_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            k = d["roofline"]["kernel_ms_per_step"]
            ks = " ".join(f"{n.replace('k_', '')} {v:.4f}" for n, v in k.items()
                          if n in ("k_search_fast", "k_esc_start", "k_search_escalated", "k_dedup", "k_emit",
                                   "k_precompute", "k_sort_scatter"))
            print(f"{f[15:-4]:10s} step {d['ms_per_step']:.4f}  {ks}")
