"""One compact line per bench_configs.py JSON line on stdin: config, alg, us per inner step, pass times."""
import json
import sys

for line in sys.stdin:
    d = json.loads(line)
    print(f"c{d['config']} {d['alg']} rho={d['rho']} {d['us_per_inner_step']:.2f} us/step "
          f"A {1e3 * d['ms_pass_a']:.1f} B {1e3 * d['ms_pass_b']:.1f}")
