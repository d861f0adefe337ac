"""Print the key numbers of bench JSON lines (tooling)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d["roofline"]
    km = r["kernel_ms_per_step"]
    print(f"{f}: value {d['value']:.3e} ms/step {d['ms_per_step']:.4f} e2e {d.get('e2e', {}).get('value', 0):.3e} "
          f"sm {d['clocks']['sm_mhz']} esc {km.get('k_esc_start', 0):.4f}+{km.get('k_search_escalated', 0):.4f} "
          f"fast {km.get('k_search_fast', 0):.4f}")
