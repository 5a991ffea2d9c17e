"""One line from a bench.py JSON line on stdin: value, graph replay, verified flags, K3 launch ms, frac."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
g = d.get("graph_replay", {})
print(d["config"]["workload"], d["value"], "graph", g.get("value"), "verified", d.get("verified"), g.get("verified"),
      "K3", d["roofline"]["launch_ms"], "frac", d["roofline"]["frac"], "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
