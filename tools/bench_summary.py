#!/usr/bin/env python3
"""One line per bench JSON line. Usage: bench_summary.py FILE... (or stdin)."""
import json
import sys


def lines():
    if len(sys.argv) > 1:
        for path in sys.argv[1:]:
            with open(path) as f:
                yield from f
    else:
        yield from sys.stdin


for line in lines():
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "config" not in d:
        print(line[:200])
        continue
    print(d["config"]["workload"][:3], d["config"].get("stream"),
          "%.4g %s" % (d["value"], d["unit"]),
          "%.3e traj-steps/s" % d.get("trajectory_steps_per_s", 0),
          "roof %.4f" % d.get("roofline", {}).get("frac", 0),
          "e2e %.3e" % d.get("e2e", {}).get("value", 0), d["config"].get("engine"), d.get("clocks"))
