"""One compact line from a bench.py JSON line on stdin: value, stream frac, ms per stream launch, SM clock."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d.get("roofline", {})
c = d.get("clocks") or {}
print(f"{d['value']:.1f} it/s frac {r.get('frac', 0):.4f} stream {1e3 * r.get('ms_per_launch', 0):.1f} us "
      f"epi {1e3 * r.get('epilogue', {}).get('ms_per_launch', 0):.1f} us sm {c.get('sm_mhz')} {c.get('reasons')}")
