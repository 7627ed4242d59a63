"""Prints the key numbers of the last bench.py JSON line of each file."""
import json
import sys

for f in sys.argv[1:]:
    lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    print(f"{f}: {d['value']:.2f} steps/s  stages {d['config'].get('stage_ms_mean')}  its {d['config'].get('pcg_iterations_mean')}"
          f"  {r.get('kernel')} {r.get('achieved', 0):.0f} GB/s frac {r.get('frac', 0):.3f} launch {r.get('avg_launch_ms', 0):.3f} ms"
          f"  clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
