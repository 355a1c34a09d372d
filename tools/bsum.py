"""One-line summaries of bench.py JSON lines: python tools/bsum.py file..."""
import json
import sys

for p in sys.argv[1:]:
    for ln in open(p):
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        r = d.get("roofline", {})
        e = d.get("e2e", {})
        print(f"{p}: {d.get('ms_per_step', 0):.4f} ms  value {d.get('value', 0):.3e}  frac {r.get('frac', 0):.3f}"
              f"  e2e {e.get('value', 0):.3e}  parity {d.get('parity')}  "
              f"lat {d.get('config', {}).get('single_batch_ms', d.get('single_sketch_ms', ''))}")
