"""Condense one bench.py JSON line (stdin) into a one-line summary."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        print(line)
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    print(f"{tag} {d['config']['workload'][:40]:40s} value={d['value']:.1f} ms/step={d['ms_per_step']*1e3:.1f}us "
          f"kernel={r.get('kernel_ms', 0)*1e3:.1f}us frac={r.get('frac', 0):.3f} clocks={d.get('clocks')}")
